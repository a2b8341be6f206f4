# round 2, GPU call 25: TMA copy with descriptor prefetch, 2x6 vs 3x4 CTA/stage configs, vs LSU
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
for c in 2d 3d; do
  timeout 120 python tools/copy_case.py $c 5 | tail -3
  CEL_COPY=tma timeout 120 python tools/copy_case.py $c 5 | tail -3
  CEL_COPY=tma CEL_TMA_CFG=1 timeout 120 python tools/copy_case.py $c 5 | tail -3
done
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 300 -k tma > gpurun_out/pytest_tma.log 2>&1; echo "tma tests rc=$?"; tail -2 gpurun_out/pytest_tma.log
