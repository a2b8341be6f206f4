# round 2, 4-GPU call 18: RSim host-cost breakdown (1 GPU vs 4 processes), with and without per-launch profiling
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
export OMP_NUM_THREADS=1
show() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step']*1e3,1), round(d['gen_us_per_step'],1), {k: round(v,1) for k,v in d['exec_us_per_step'].items()}, {k: round(v,1) for k,v in d['host_us_per_step'].items()}, {k: round(v,2) for k,v in d['per_step'].items()})"; }
CEL_BENCH_NOPROF=1 timeout 300 python bench_config.py --workload rsim --gpus 1 > gpurun_out/r1g.json 2> gpurun_out/r1g.err; echo "rsim 1 GPU noprof rc=$?"; show gpurun_out/r1g.json
for P in 1 0; do
  if [ $P = 1 ]; then E=""; else E="CEL_BENCH_NOPROF=1"; fi
  env $E timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2991$P bench_config.py --workload rsim --gpus 4 > gpurun_out/r4_$P.json 2> gpurun_out/r4_$P.err
  echo "rsim 4 processes prof=$P rc=$?"; show gpurun_out/r4_$P.json
done
CEL_BENCH_NOPROF=1 CEL_SCHED_MEMO=0 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29920 bench_config.py --workload rsim --gpus 4 > gpurun_out/r4_nm.json 2> gpurun_out/r4_nm.err
echo "rsim 4 processes noprof nomemo rc=$?"; show gpurun_out/r4_nm.json
CEL_BENCH_NOPROF=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29921 bench_config.py --workload rsim --gpus 4 --lookahead none > gpurun_out/r4_none.json 2> gpurun_out/r4_none.err
echo "rsim 4 processes lookahead none rc=$?"; show gpurun_out/r4_none.json
