# round 2, 4-GPU call 32: coalesced free ranges fold long tokens into one event -- suite, mp_check, RSim lookahead none
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
export OMP_NUM_THREADS=1
timeout 1500 python -m pytest tests -m gpu -q --timeout 400 --timeout-method thread > gpurun_out/pytest4.log 2>&1
echo "pytest all (4 GPUs) rc=$?"; tail -2 gpurun_out/pytest4.log; grep -E "^E |^FAILED" gpurun_out/pytest4.log | head -20
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 600 $TR --master-port 29604 tests/mp_check.py --execute 1 > gpurun_out/mp_all4.log 2>&1
echo "mp_check all N=4 rc=$?"; grep -E "FAIL|MP_CHECK" gpurun_out/mp_all4.log | tail -2
show() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step']*1e3,1), {k: round(v,1) for k,v in d['exec_us_per_step'].items()})"; }
CEL_BENCH_NOPROF=1 timeout 600 $TR --master-port 29921 bench_config.py --workload rsim --gpus 4 --lookahead none > gpurun_out/r4_none.json 2> gpurun_out/r4_none.err; echo "rsim 4p none rc=$?"; show gpurun_out/r4_none.json
CEL_BENCH_NOPROF=1 timeout 600 $TR --master-port 29922 bench_config.py --workload rsim --gpus 4 > gpurun_out/r4_auto.json 2> gpurun_out/r4_auto.err; echo "rsim 4p auto rc=$?"; show gpurun_out/r4_auto.json
CEL_BENCH_NOPROF=1 timeout 300 python bench_config.py --workload rsim --gpus 1 --lookahead none > gpurun_out/r1_none.json 2> gpurun_out/r1_none.err; echo "rsim 1 GPU none rc=$?"; show gpurun_out/r1_none.json
