# round 2, GPU call 27: wave5 with programmatic dependent launch: parity + bench A/B
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 300 --timeout-method thread -k "wavesim or smoke" > gpurun_out/pytest_w.log 2>&1
echo "wavesim tests rc=$?"; tail -2 gpurun_out/pytest_w.log; grep -E "^E |^FAILED" gpurun_out/pytest_w.log | head
for p in 1 0 1 0; do CEL_PDL=$p timeout 300 python bench.py --steps 2000 --warmup 20 --no-e2e --no-cpu-baseline --no-copy > gpurun_out/b.json 2>&1; echo "bench pdl=$p"; python -c "
import json; d=json.loads(open('gpurun_out/b.json').read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'], d['roofline']['kernel_share_of_step'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"; done
