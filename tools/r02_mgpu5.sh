# round 2, 4-GPU call 5: receiver-only member tokens; RSim fused rows in 1 and 4 processes; suite
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
j() { python -c "
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
keys=('value','ms_per_step','gen_us_per_step','exec_us_per_step','coll_groups','coll_p2p','coll_fused','GBps_received_per_device')
print({k: d.get(k) for k in keys}, {k: v for k, v in d.get('profile_ms', {}).items() if k in ('coll','rsim_row')})" $1; }
for f in 1 0; do
  CEL_FUSE_ROWS=$f timeout 300 python bench_config.py --workload rsim --gpus 4 > gpurun_out/r1_f$f.json 2> gpurun_out/r1_f$f.err
  echo "rsim 4 GPUs 1 process fuse=$f rc=$?"; j gpurun_out/r1_f$f.json
  CEL_FUSE_ROWS=$f timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2963$f bench_config.py --workload rsim --gpus 4 > gpurun_out/r4_f$f.json 2> gpurun_out/r4_f$f.err
  echo "rsim 4 processes fuse=$f rc=$?"; j gpurun_out/r4_f$f.json
  CEL_FUSE_ROWS=$f timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2964$f bench_config.py --workload rsim --gpus 2 > gpurun_out/r2_f$f.json 2> gpurun_out/r2_f$f.err
  echo "rsim 2 processes fuse=$f rc=$?"; j gpurun_out/r2_f$f.json
done
CEL_COLL_P2P=0 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29650 bench_config.py --workload rsim --gpus 4 > gpurun_out/r4_push.json 2> gpurun_out/r4_push.err
echo "rsim 4 processes pushes rc=$?"; j gpurun_out/r4_push.json
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29651 bench_config.py --workload gather --gpus 4 > gpurun_out/g4.json 2> gpurun_out/g4.err
echo "gather 4 processes P2P rc=$?"; j gpurun_out/g4.json
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 --timeout-method thread > gpurun_out/pytest.log 2>&1
echo "pytest all rc=$?"; tail -3 gpurun_out/pytest.log; grep -E "^E |^FAILED" gpurun_out/pytest.log | head -20
