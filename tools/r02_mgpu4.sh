# round 2, 4-GPU call 4: suite (P2P + fused rows in one process), WaveSim N=2/4 with 8-row strips, RSim single process fused
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 --timeout-method thread > gpurun_out/pytest.log 2>&1
echo "pytest all rc=$?"; tail -3 gpurun_out/pytest.log; grep -E "^E |^FAILED" gpurun_out/pytest.log | head -20
j() { python -c "
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
keys=('value','ms_per_step','gen_us_per_step','exec_us_per_step','coll_groups','coll_p2p','coll_fused','GBps_received_per_device')
print({k: d.get(k) for k in keys}, {k: v for k, v in d.get('profile_ms', {}).items() if k in ('coll','rsim_row')})" $1; }
for f in 1 0; do
  CEL_FUSE_ROWS=$f timeout 300 python bench_config.py --workload rsim --gpus 4 > gpurun_out/r1_f$f.json 2> gpurun_out/r1_f$f.err
  echo "rsim 4 GPUs 1 process fuse=$f rc=$?"; j gpurun_out/r1_f$f.json
  CEL_FUSE_ROWS=$f timeout 300 python bench_config.py --workload rsim --gpus 2 > gpurun_out/r1b_f$f.json 2> gpurun_out/r1b_f$f.err
  echo "rsim 2 GPUs 1 process fuse=$f rc=$?"; j gpurun_out/r1b_f$f.json
done
timeout 300 python bench_config.py --workload rsim --gpus 1 > gpurun_out/r1c.json 2> gpurun_out/r1c.err; echo "rsim 1 GPU"; j gpurun_out/r1c.json
for N in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2960$N bench.py --gpus $N --steps 1000 --warmup 20 --no-e2e > gpurun_out/bench_n$N.json 2> gpurun_out/bench_n$N.err
  echo "bench N=$N rc=$?"; python -c "import json; d=json.loads(open('gpurun_out/bench_n$N.json').read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'], d['roofline']['kernel_share_of_step'], d['clocks'], d['host_submit_us_per_step'])"
done
timeout 600 python bench.py --gpus 1 --steps 1000 --warmup 20 --no-e2e --no-cpu-baseline --no-copy > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err
echo "bench N=1 rc=$?"; python -c "import json; d=json.loads(open('gpurun_out/bench_n1.json').read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'], d['clocks'])"
