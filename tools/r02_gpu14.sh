# round 2, GPU call 14: wave5 strip sweep, suite refresh, ncu of the copy kernels (LSU vs TMA) and the bench launch list
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 --timeout-method thread > gpurun_out/pytest.log 2>&1
echo "pytest all rc=$?"; tail -4 gpurun_out/pytest.log; grep -E "^E |^FAILED" gpurun_out/pytest.log | head -20
for rows in 16384 8192 4096 2048; do
  for h in 0 6 8 12 16 24 32; do
    if [ $h = 0 ]; then timeout 120 python tools/wave_strip.py $rows; else CEL_WAVE_STRIP=$h timeout 120 python tools/wave_strip.py $rows; fi
  done
done 2>&1 | grep rows
timeout 900 python bench_suite.py --out gpurun_out/r02_suite.json > gpurun_out/suite.log 2>&1; echo "suite rc=$?"; tail -c 1500 gpurun_out/suite.log
timeout 120 python tools/copy_case.py 2d && CEL_COPY=tma timeout 120 python tools/copy_case.py 2d && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"copy_kernel" -s 2 -c 2 -o gpurun_out/ncu_copy2d_lsu python tools/copy_case.py 2d > gpurun_out/ncu_copy_lsu.log 2>&1
echo "ncu lsu rc=$?"
CEL_COPY=tma timeout 600 ncu --set full --clock-control none --import-source on -k regex:"copy_kernel_tmap" -s 1 -c 1 -o gpurun_out/ncu_copy2d_tma python tools/copy_case.py 2d > gpurun_out/ncu_copy_tma.log 2>&1
echo "ncu tma rc=$?"
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-copy --no-e2e > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches_wavesim_n1.csv python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-copy --no-e2e > gpurun_out/ncu_launch.log 2>&1
echo "ncu launches rc=$?"
