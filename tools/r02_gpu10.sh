# round 2, GPU call 10: device-direct sends (virtual-node mode), VMM test fix, whole suite
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_cluster.py tests/test_gpu_parity.py -m gpu -q -x --timeout 600 -k "direct or vmm or overflow" > gpurun_out/pytest_new.log 2>&1
echo "pytest new rc=$?"; tail -30 gpurun_out/pytest_new.log
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest.log 2>&1
echo "pytest all rc=$?"; tail -6 gpurun_out/pytest.log
