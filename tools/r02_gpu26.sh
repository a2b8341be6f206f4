# round 2, GPU call 26: scheduler compile memo -- 1-GPU suite, bench line, host cost on the box's CPU
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests -m gpu -q --timeout 300 --timeout-method thread > gpurun_out/pytest1.log 2>&1
echo "pytest -m gpu rc=$?"; tail -2 gpurun_out/pytest1.log; grep -E "^E |^FAILED" gpurun_out/pytest1.log | head -20
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_k20.json 2> gpurun_out/bench_k20.err
echo "bench rc=$?"; tail -1 gpurun_out/bench_k20.json | cut -c1-400
timeout 300 python tools/sched_cost.py > gpurun_out/sched_cost.txt 2>&1; cat gpurun_out/sched_cost.txt
CEL_SCHED_MEMO=0 timeout 300 python tools/sched_cost.py > gpurun_out/sched_cost_nomemo.txt 2>&1; cat gpurun_out/sched_cost_nomemo.txt
g++ -O2 -std=c++17 -Ipaper_2503_10516_b200/csrc tools/sched_prof.cpp paper_2503_10516_b200/csrc/sched.cpp paper_2503_10516_b200/csrc/sched_memo.cpp -o /tmp/sched_prof && for g in 4 8; do /tmp/sched_prof $g 0 20000; CEL_SCHED_MEMO=0 /tmp/sched_prof $g 0 5000; done; /tmp/sched_prof rsim 4 0; /tmp/sched_prof rsim 1
nproc; lscpu | grep -E "Model name|MHz" | head -3
