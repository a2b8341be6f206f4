# round 2, GPU call 11: device-direct sends after the deadlock fix (short timeouts), then the whole suite
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 400 python -m pytest tests/test_gpu_cluster.py -m gpu -q -x --timeout 180 --timeout-method thread -k "direct" > gpurun_out/pytest_direct.log 2>&1
echo "pytest direct rc=$?"; tail -30 gpurun_out/pytest_direct.log
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 300 --timeout-method thread -k "vmm or overflow" > gpurun_out/pytest_vmm.log 2>&1
echo "pytest vmm rc=$?"; tail -15 gpurun_out/pytest_vmm.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 --timeout-method thread > gpurun_out/pytest.log 2>&1
echo "pytest all rc=$?"; tail -6 gpurun_out/pytest.log
