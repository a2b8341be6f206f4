# round 2, 4-GPU call 29: RSim row chain (re-applied) -- full 4-GPU suite, mp_check at 2 / 4, RSim at 4 / 2 / 1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
export OMP_NUM_THREADS=1
timeout 1500 python -m pytest tests -m gpu -q --timeout 400 --timeout-method thread > gpurun_out/pytest4.log 2>&1
echo "pytest all (4 GPUs) rc=$?"; tail -2 gpurun_out/pytest4.log; grep -E "^E |^FAILED" gpurun_out/pytest4.log | head -20
for N in 2 4; do
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
timeout 600 $TR --master-port 2960$N tests/mp_check.py --execute 1 > gpurun_out/mp_all$N.log 2>&1
echo "mp_check all N=$N rc=$?"; grep -E "FAIL|MP_CHECK|chained" gpurun_out/mp_all$N.log | tail -3
done
show() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step']*1e3,1), round(d['gen_us_per_step'],1), {k: round(v,1) for k,v in d['exec_us_per_step'].items()})"; }
for N in 4 2; do
CEL_BENCH_NOPROF=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2991$N bench_config.py --workload rsim --gpus $N > gpurun_out/r${N}.json 2> gpurun_out/r${N}.err; echo "rsim ${N}p rc=$?"; show gpurun_out/r${N}.json
done
CEL_BENCH_NOPROF=1 timeout 300 python bench_config.py --workload rsim --gpus 1 > gpurun_out/r1g.json 2> gpurun_out/r1g.err; echo "rsim 1 GPU rc=$?"; show gpurun_out/r1g.json
