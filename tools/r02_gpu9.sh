# round 2, GPU call 9: hybrid arena / VMM placement; whole -m gpu suite; bench line
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest.log 2>&1
echo "pytest all rc=$?"; tail -6 gpurun_out/pytest.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_k20.json 2> gpurun_out/bench_k20.err
echo "bench rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/bench_k20.json'))
print(d['value'], d['roofline']['frac'], d['e2e']['value'], d['clocks'])"
