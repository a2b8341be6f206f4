# round 2, GPU call 28: whole suite with PDL kernels (1 GPU), smoke, driver bench line
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 --timeout-method thread > gpurun_out/pytest.log 2>&1
echo "pytest all rc=$?"; tail -3 gpurun_out/pytest.log; grep -E "^E |^FAILED" gpurun_out/pytest.log | head -20
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"; echo "smoke rc=$?"
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_k20.json 2> gpurun_out/bench_k20.err; echo "bench k20 rc=$?"; cat gpurun_out/bench_k20.json | head -c 1500
