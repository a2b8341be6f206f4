# round 2, 4-GPU call 26: RSim fused rows wait for the incoming rows only before their stage -- parity, bench, trace
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
export OMP_NUM_THREADS=1
for N in 2 4; do
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
timeout 300 $TR --master-port 2960$N tests/mp_check.py --execute 1 --quick --only rsim > gpurun_out/mp_rsim$N.log 2>&1
echo "mp_check rsim N=$N rc=$?"; grep -E "FAIL|MP_CHECK" gpurun_out/mp_rsim$N.log | tail -2
done
show() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step']*1e3,1), {k: (round(v['ms'],2), v['launches']) for k,v in d['profile_ms'].items()})"; }
for N in 4 2; do
CEL_BENCH_NOPROF=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2991$N bench_config.py --workload rsim --gpus $N > gpurun_out/r${N}_n.json 2> gpurun_out/r${N}_n.err; echo "rsim ${N}p noprof rc=$?"; show gpurun_out/r${N}_n.json
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2992$N bench_config.py --workload rsim --gpus $N > gpurun_out/r${N}_p.json 2> gpurun_out/r${N}_p.err; echo "rsim ${N}p prof rc=$?"; show gpurun_out/r${N}_p.json
done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29950 tools/trace_rsim.py > gpurun_out/trace_rsim.log 2>&1; echo "trace rc=$?"; tail -12 gpurun_out/trace_rsim.log
