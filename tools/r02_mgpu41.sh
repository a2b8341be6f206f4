# round 2, 4-GPU call 41: executor hand-off as a ring of reused slots -- suite on 4 GPUs, mp_check, RSim, WaveSim
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
export OMP_NUM_THREADS=1
timeout 1500 python -m pytest tests -m gpu -q --timeout 400 --timeout-method thread > gpurun_out/pytest4.log 2>&1
echo "pytest all (4 GPUs) rc=$?"; tail -2 gpurun_out/pytest4.log; grep -E "^E |^FAILED" gpurun_out/pytest4.log | head -20
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 600 $TR --master-port 29604 tests/mp_check.py --execute 1 > gpurun_out/mp_all4.log 2>&1
echo "mp_check all N=4 rc=$?"; grep -E "FAIL|MP_CHECK" gpurun_out/mp_all4.log | tail -2
show() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step']*1e3,1), round(d['gen_us_per_step'],1), {k: round(v,1) for k,v in d['exec_us_per_step'].items()})"; }
for N in 4 2; do
CEL_BENCH_NOPROF=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2991$N bench_config.py --workload rsim --gpus $N > gpurun_out/rs$N.json 2> gpurun_out/rs$N.err; echo "rsim ${N}p rc=$?"; show gpurun_out/rs$N.json
done
CEL_BENCH_NOPROF=1 timeout 300 python bench_config.py --workload rsim --gpus 1 > gpurun_out/rs1.json 2> gpurun_out/rs1.err; echo "rsim 1 GPU rc=$?"; show gpurun_out/rs1.json
timeout 600 python bench.py --steps 1000 --warmup 20 --no-e2e --no-cpu-baseline --no-copy > gpurun_out/b1.json 2> gpurun_out/b1.err
echo "bench N=1 rc=$?"; tail -1 gpurun_out/b1.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'])"
timeout 600 $TR --master-port 29940 bench.py --gpus 4 --steps 1000 --warmup 20 --no-e2e > gpurun_out/b4.json 2> gpurun_out/b4.err
echo "bench N=4 rc=$?"; tail -1 gpurun_out/b4.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'])"
