# round 2, GPU call 26: programmatic dependent launch for RSim rows: parity + A/B
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 300 --timeout-method thread -k "rsim" > gpurun_out/pytest_rsim.log 2>&1
echo "rsim tests rc=$?"; tail -2 gpurun_out/pytest_rsim.log; grep -E "^E |^FAILED" gpurun_out/pytest_rsim.log | head
for p in 1 0 1 0; do CEL_PDL=$p timeout 300 python bench_config.py --workload rsim --gpus 1 > gpurun_out/rs.json 2>&1; echo "rsim 1 GPU pdl=$p"; python -c "
import json; d=json.loads(open('gpurun_out/rs.json').read().strip().splitlines()[-1]); print(d['value'], d['profile_ms'])"; done
for p in 1 0; do CEL_PDL=$p CEL_NO_GROW=0 timeout 300 python bench_config.py --workload rsim --gpus 1 --lookahead none > gpurun_out/rs.json 2>&1; echo "rsim none 1 GPU pdl=$p"; python -c "
import json; d=json.loads(open('gpurun_out/rs.json').read().strip().splitlines()[-1]); print(d['value'])"; done
