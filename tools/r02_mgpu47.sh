# round 2, 4-GPU call 47: hand-off ring with batch claims (CEL_EXEC_RING=1) vs the deque -- RSim A/B, parity
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
export OMP_NUM_THREADS=1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
CEL_EXEC_RING=1 timeout 600 $TR --master-port 29604 tests/mp_check.py --execute 1 --quick > gpurun_out/mp_ring.log 2>&1
echo "mp_check ring rc=$?"; grep -E "FAIL|MP_CHECK" gpurun_out/mp_ring.log | tail -2
show() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step']*1e3,1))"; }
for R in 1 0 1 0; do
  for N in 4 2; do
    CEL_EXEC_RING=$R CEL_BENCH_NOPROF=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2991$N bench_config.py --workload rsim --gpus $N > gpurun_out/rs.json 2> gpurun_out/rs.err
    echo "rsim ${N}p ring=$R rc=$?"; show gpurun_out/rs.json
  done
done
CEL_EXEC_RING=1 timeout 600 $TR --master-port 29940 bench.py --gpus 4 --steps 1000 --warmup 20 --no-e2e > gpurun_out/b4.json 2> gpurun_out/b4.err
echo "bench N=4 ring rc=$?"; tail -1 gpurun_out/b4.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'])"
