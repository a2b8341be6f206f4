# round 2, GPU call 15: strip 8, P2P gathers on one GPU (suite), copy timing LSU vs TMA, bench N=1, ncu
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 --timeout-method thread > gpurun_out/pytest.log 2>&1
echo "pytest all rc=$?"; tail -3 gpurun_out/pytest.log; grep -E "^E |^FAILED" gpurun_out/pytest.log | head -20
for c in 2d 3d 1g; do timeout 120 python tools/copy_case.py $c 4 | tail -2; CEL_COPY=tma timeout 120 python tools/copy_case.py $c 4 | tail -2; done
timeout 600 python bench.py --steps 2000 --warmup 20 > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err
echo "bench rc=$?"; cat gpurun_out/bench_n1.json
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-copy --no-e2e > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches_wavesim_n1.csv python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-copy --no-e2e > gpurun_out/ncu_launch.log 2>&1
echo "ncu launches rc=$?"
timeout 120 python tools/copy_case.py 2d 2 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"copy_kernel" -s 1 -c 1 -o gpurun_out/ncu_copy2d_lsu python tools/copy_case.py 2d 2 > gpurun_out/ncu_copy_lsu.log 2>&1
echo "ncu lsu rc=$?"
timeout 300 python tools/wave_strip.py 16384 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"wave5" -s 30 -c 1 -o gpurun_out/ncu_wave5_h8 python tools/wave_strip.py 16384 > gpurun_out/ncu_wave5.log 2>&1
echo "ncu wave5 rc=$?"
