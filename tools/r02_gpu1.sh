# round 2, GPU call 1: build, -m gpu suite (minus the folded multi-process test), bench lines
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 -k "not multiprocess_gpu" > gpurun_out/pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest.log
tail -30 gpurun_out/pytest.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_k20.json 2> gpurun_out/bench_k20.err
echo "bench k20 rc=$?"; cat gpurun_out/bench_k20.json | head -c 6000
timeout 900 python bench.py --no-cpu-baseline --no-copy > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
echo "bench default rc=$?"; head -c 3000 gpurun_out/bench_default.json
