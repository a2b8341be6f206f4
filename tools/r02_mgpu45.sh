# round 2, 2-GPU call 45: after the trap-threshold change -- smoke, multi-process parity (fused paths)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
export OMP_NUM_THREADS=1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 900 python -m pytest tests/test_multiprocess.py -m gpu -q --timeout 400 --timeout-method thread > gpurun_out/pytest_mp.log 2>&1
echo "multiprocess tests rc=$?"; tail -2 gpurun_out/pytest_mp.log
