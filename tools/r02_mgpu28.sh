# round 2, 4-GPU call 28: RSim row chain (next row waits for the previous row's local stores, not its grid)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
export OMP_NUM_THREADS=1
for N in 2 4; do
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
timeout 600 $TR --master-port 2960$N tests/mp_check.py --execute 1 > gpurun_out/mp_all$N.log 2>&1
echo "mp_check all N=$N rc=$?"; grep -E "FAIL|MP_CHECK|chained" gpurun_out/mp_all$N.log | tail -4
done
show() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step']*1e3,1), {k: (round(v['ms'],2), v['launches']) for k,v in d['profile_ms'].items()})"; }
for C in 1 0; do
CEL_RSIM_CHAIN=$C CEL_BENCH_NOPROF=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2991$C bench_config.py --workload rsim --gpus 4 > gpurun_out/r4_c$C.json 2> gpurun_out/r4_c$C.err; echo "rsim 4p chain=$C rc=$?"; show gpurun_out/r4_c$C.json
done
CEL_BENCH_NOPROF=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29922 bench_config.py --workload rsim --gpus 2 > gpurun_out/r2_c1.json 2> gpurun_out/r2_c1.err; echo "rsim 2p chain rc=$?"; show gpurun_out/r2_c1.json
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29950 tools/trace_rsim.py > gpurun_out/trace_rsim.log 2>&1; echo "trace rc=$?"; tail -8 gpurun_out/trace_rsim.log
