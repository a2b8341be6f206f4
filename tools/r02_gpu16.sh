# round 2, GPU call 16: RSim rows fused with their gathers; P2P gathers; whole suite
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 240 --timeout-method thread -k "fused or rsim" > gpurun_out/pytest_fuse.log 2>&1
echo "pytest fuse rc=$?"; grep -E "^E |passed|failed|Timeout" gpurun_out/pytest_fuse.log | head -20
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 --timeout-method thread > gpurun_out/pytest.log 2>&1
echo "pytest all rc=$?"; tail -3 gpurun_out/pytest.log; grep -E "^E |^FAILED" gpurun_out/pytest.log | head -20
for f in 1 0; do CEL_FUSE_ROWS=$f timeout 300 python bench_config.py --workload rsim --gpus 1 > gpurun_out/rsim1_f$f.json 2>&1; echo "rsim 1 GPU fuse=$f"; tail -c 600 gpurun_out/rsim1_f$f.json; echo; done
