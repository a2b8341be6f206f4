# round 2, 4-GPU call 33: elided resize copies fold long tokens -- RSim lookahead none at 4 processes, parity
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
export OMP_NUM_THREADS=1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
show() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step']*1e3,1), {k: round(v,1) for k,v in d['exec_us_per_step'].items()})"; }
CEL_BENCH_NOPROF=1 timeout 600 $TR --master-port 29921 bench_config.py --workload rsim --gpus 4 --lookahead none > gpurun_out/r4_none.json 2> gpurun_out/r4_none.err; echo "rsim 4p none rc=$?"; show gpurun_out/r4_none.json
timeout 600 $TR --master-port 29604 tests/mp_check.py --execute 1 > gpurun_out/mp_all4.log 2>&1
echo "mp_check all N=4 rc=$?"; grep -E "FAIL|MP_CHECK" gpurun_out/mp_all4.log | tail -2
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_multiprocess.py -m gpu -q --timeout 400 --timeout-method thread > gpurun_out/pytest_p.log 2>&1
echo "parity + multiprocess rc=$?"; tail -2 gpurun_out/pytest_p.log
