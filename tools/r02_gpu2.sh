# round 2, GPU call 2: TMA tensor-map copies, bench copy block A/B, folded multi-process test (last: it may hang)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 600 -k "tma_tensor_map" > gpurun_out/pytest_tma.log 2>&1
echo "pytest tma rc=$?"; tail -15 gpurun_out/pytest_tma.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_copy.json 2> gpurun_out/bench_copy.err
echo "bench rc=$?"; python -c "import json; d=json.load(open('gpurun_out/bench_copy.json')); print(json.dumps(d['copy'], indent=1))"
timeout 400 python -m pytest tests/test_multiprocess.py -m gpu -q --timeout 380 > gpurun_out/pytest_mp.log 2>&1
echo "pytest mp rc=$?"; tail -30 gpurun_out/pytest_mp.log
