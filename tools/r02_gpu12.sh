# round 2, GPU call 12: device-direct sends (opt-in) on the configs, then the whole suite
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 400 python -m pytest tests/test_gpu_cluster.py -m gpu -q --timeout 180 --timeout-method thread -k "direct" > gpurun_out/pytest_direct.log 2>&1
echo "pytest direct rc=$?"; tail -30 gpurun_out/pytest_direct.log | grep -v "^ "
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 --timeout-method thread > gpurun_out/pytest.log 2>&1
echo "pytest all rc=$?"; tail -6 gpurun_out/pytest.log
