# round 2, GPU call 5: TMA column boxes after the tile-width guard; row padding and VMM A/B on the copy block
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
export CUDA_LAUNCH_BLOCKING=1 CEL_EXEC_THREAD=0
for c in "ws2d_axes 4" "ws2d_box 4 none" "rand1 4 none" "rand4 4 none" "rand5 3 none" "rand6 4 auto" "rand7 4 none"; do
  CEL_COPY=tma CEL_NO_GROW=1 timeout 120 python tests/tools/tma_debug.py $c 2>&1 | tail -1
done
unset CUDA_LAUNCH_BLOCKING CEL_EXEC_THREAD
for cfg in "CEL_ROW_ALIGN=16" "CEL_ROW_ALIGN=128" "CEL_ROW_ALIGN=128 CEL_NO_VMM=1"; do
  env $cfg timeout 600 python bench.py --steps 200 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_ab.json 2> gpurun_out/bench_ab.err
  echo "$cfg rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/bench_ab.json'))
print(d['value'], d['roofline']['frac'], d['roofline']['kernel_share_of_step'])
for k,v in d['copy'].items(): print(' ', k, v.get('GBps_hbm_rw'), v.get('frac_hbm'), v.get('us_per_copy'), v.get('bytes_ok'), v.get('kernel'))"
done
