# round 2, 4-GPU call 8: shells on the compute stream (A/B) at N=2/4; Fig. 7-style timeline at N=4
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
for N in 4 2; do
  for sc in 0 1 0 1; do
    CEL_SHELL_ON_COMPUTE=$sc timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2980$N bench.py --gpus $N --steps 1000 --warmup 20 --no-e2e > gpurun_out/bench_sc.json 2> gpurun_out/bench_sc.err
    echo "bench N=$N shell_on_compute=$sc rc=$?"; tail -1 gpurun_out/bench_sc.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['roofline']['kernel_share_of_step'], d['clocks']['reasons'])"
  done
done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29811 tools/trace_wavesim.py > gpurun_out/trace.log 2>&1; echo "trace rc=$?"; tail -8 gpurun_out/trace.log
