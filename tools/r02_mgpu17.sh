# round 2, 4-GPU call 17: fused halo default on -- full GPU suite on 4 GPUs, bench N=1..4, timeline
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
export OMP_NUM_THREADS=1
timeout 1500 python -m pytest tests -m gpu -q --timeout 400 --timeout-method thread > gpurun_out/pytest4.log 2>&1
echo "pytest all (4 GPUs) rc=$?"; tail -2 gpurun_out/pytest4.log; grep -E "^E |^FAILED" gpurun_out/pytest4.log | head -20
timeout 600 python bench.py --steps 1000 --warmup 20 --no-e2e --no-cpu-baseline --no-copy > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err
echo "bench N=1 rc=$?"; tail -1 gpurun_out/bench_n1.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['clocks'])"
for N in 2 3 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2990$N bench.py --gpus $N --steps 1000 --warmup 20 > gpurun_out/bench_n$N.json 2> gpurun_out/bench_n$N.err
  echo "bench N=$N rc=$?"; tail -1 gpurun_out/bench_n$N.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['roofline']['kernel_share_of_step'], d['clocks']['reasons'], d['e2e']['value'] if d.get('e2e') else None, d.get('halo_fused_per_step'))"
done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29650 tools/trace_wavesim.py > gpurun_out/trace_fused4.log 2>&1; echo "trace rc=$?"; tail -6 gpurun_out/trace_fused4.log
