# ncu --set full of one peer push (1 GiB 'all' read between 2 GPUs: 512 MiB per direction)
python - <<'PY' > gpurun_out/peer_prog.log 2>&1
import sys, os
sys.path.insert(0, os.getcwd())
from paper_2503_10516_b200 import cel
N = (1 << 30) // 16
rt = cel.Runtime(2, cuda_devices=[0, 1], arena_bytes=3 << 30, collective=False)
rt.buffer_create(1, [N], 16); rt.buffer_create(1, [N], 16)
rt.task_submit({"dims": 1, "range": ([0], [N]), "kernel": "fill_const", "params": {"value": 1.0}, "accesses": [(0, "write", ("one_to_one",))]})
rt.wait()
rt.task_submit({"dims": 1, "range": ([0], [N]), "kernel": "fill_const", "params": {"value": 2.0}, "accesses": [(0, "read", ("all",)), (1, "write", ("one_to_one",))]})
rt.wait()
rt.shutdown()
print("ok")
PY
cat gpurun_out/peer_prog.log
cat > /tmp/peer.py <<'PY'
import sys, os
sys.path.insert(0, os.environ["GRAFT_REPO_ROOT"] if "GRAFT_REPO_ROOT" in os.environ else os.getcwd())
from paper_2503_10516_b200 import cel
N = (1 << 30) // 16
rt = cel.Runtime(2, cuda_devices=[0, 1], arena_bytes=3 << 30, collective=False)
rt.buffer_create(1, [N], 16); rt.buffer_create(1, [N], 16)
rt.task_submit({"dims": 1, "range": ([0], [N]), "kernel": "fill_const", "params": {"value": 1.0}, "accesses": [(0, "write", ("one_to_one",))]})
rt.wait()
rt.task_submit({"dims": 1, "range": ([0], [N]), "kernel": "fill_const", "params": {"value": 2.0}, "accesses": [(0, "read", ("all",)), (1, "write", ("one_to_one",))]})
rt.wait()
rt.shutdown()
PY
timeout 500 ncu --set full --clock-control none -k regex:copy_kernel --launch-skip 2 --launch-count 1 -o gpurun_out/peer_push2 python /tmp/peer.py > gpurun_out/ncu_peer.log 2>&1
tail -3 gpurun_out/ncu_peer.log
