# round 2, 4-GPU call 24: validation after the scheduler changes + RSim host-side experiments
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
export OMP_NUM_THREADS=1
lscpu -e | head -20
timeout 1500 python -m pytest tests -m gpu -q --timeout 400 --timeout-method thread > gpurun_out/pytest4.log 2>&1
echo "pytest all (4 GPUs) rc=$?"; tail -2 gpurun_out/pytest4.log; grep -E "^E |^FAILED" gpurun_out/pytest4.log | head -20
show() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step']*1e3,1), round(d['gen_us_per_step'],1), {k: round(v,1) for k,v in d['exec_us_per_step'].items()}, {k: round(v,2) for k,v in d['per_step'].items()})"; }
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
CEL_BENCH_NOPROF=1 timeout 300 $TR --master-port 29911 bench_config.py --workload rsim --gpus 4 > gpurun_out/r4_a.json 2> gpurun_out/r4_a.err; echo "rsim 4p default rc=$?"; show gpurun_out/r4_a.json
CEL_BENCH_NOPROF=1 CEL_PIN=0 timeout 300 $TR --master-port 29912 bench_config.py --workload rsim --gpus 4 > gpurun_out/r4_b.json 2> gpurun_out/r4_b.err; echo "rsim 4p nopin rc=$?"; show gpurun_out/r4_b.json
CEL_BENCH_NOPROF=1 timeout 300 $TR --master-port 29913 bench_config.py --workload rsim --gpus 4 > gpurun_out/r4_c.json 2> gpurun_out/r4_c.err; echo "rsim 4p default again rc=$?"; show gpurun_out/r4_c.json
CEL_BENCH_NOPROF=1 timeout 300 python bench_config.py --workload rsim --gpus 1 > gpurun_out/r1g.json 2> gpurun_out/r1g.err; echo "rsim 1 GPU rc=$?"; show gpurun_out/r1g.json
g++ -O2 -std=c++17 -Ipaper_2503_10516_b200/csrc tools/sched_prof.cpp paper_2503_10516_b200/csrc/sched.cpp paper_2503_10516_b200/csrc/sched_memo.cpp -o /tmp/sched_prof && /tmp/sched_prof rsim 4 0 && /tmp/sched_prof rsim 2 0 && /tmp/sched_prof 8 0 20000
timeout 300 python tools/sched_cost.py
