# round 2, GPU call 3: TMA copies (fixed), VMM allocations, the whole -m gpu suite, bench
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 500 -k "tma_tensor_map or vmm" > gpurun_out/pytest_new.log 2>&1
echo "pytest new rc=$?"; tail -25 gpurun_out/pytest_new.log
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest.log 2>&1
echo "pytest all rc=$?"; tail -8 gpurun_out/pytest.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_copy.json 2> gpurun_out/bench_copy.err
echo "bench rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/bench_copy.json'))
print(d['value'], d['roofline']['frac'])
for k,v in d['copy'].items(): print(k, v.get('GBps_hbm_rw'), v.get('frac_hbm'), v.get('us_per_copy'), v.get('bytes_ok'), v.get('kernel'))"
