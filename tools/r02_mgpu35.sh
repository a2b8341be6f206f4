# round 2, 4-GPU call 35: final lines after the wave5 variant rule -- suite on 4 GPUs, bench N=1..4, RSim 4/2/1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
export OMP_NUM_THREADS=1
timeout 1500 python -m pytest tests -m gpu -q --timeout 400 --timeout-method thread > gpurun_out/pytest4.log 2>&1
echo "pytest all (4 GPUs) rc=$?"; tail -2 gpurun_out/pytest4.log; grep -E "^E |^FAILED" gpurun_out/pytest4.log | head -20
timeout 900 python bench.py > gpurun_out/final_n1_default.json 2> gpurun_out/final_n1_default.err
echo "bench default rc=$?"; tail -1 gpurun_out/final_n1_default.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['e2e']['value'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
for N in 2 3 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2990$N bench.py --gpus $N --steps 1000 --warmup 20 > gpurun_out/final_n$N.json 2> gpurun_out/final_n$N.err
  echo "bench N=$N rc=$?"; tail -1 gpurun_out/final_n$N.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['kernel'], d['roofline']['frac'], d['roofline']['kernel_share_of_step'], d['clocks']['reasons'], d['e2e']['value'] if d.get('e2e') else None)"
done
show() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step']*1e3,1))"; }
for N in 4 2; do
CEL_BENCH_NOPROF=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2991$N bench_config.py --workload rsim --gpus $N > gpurun_out/final_rsim$N.json 2> gpurun_out/final_rsim$N.err; echo "rsim ${N}p rc=$?"; show gpurun_out/final_rsim$N.json
done
CEL_BENCH_NOPROF=1 timeout 300 python bench_config.py --workload rsim --gpus 1 > gpurun_out/final_rsim1.json 2> gpurun_out/final_rsim1.err; echo "rsim 1 GPU rc=$?"; show gpurun_out/final_rsim1.json
