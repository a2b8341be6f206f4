# round 2, GPU call 4: locate the illegal instruction (one program per process), VMM A/B, TMA copy A/B
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
export CUDA_LAUNCH_BLOCKING=1 CEL_EXEC_THREAD=0
for c in "jac36 4" "jac20 5" "ws2d_axes 2" "ws2d_axes 4" "ws2d_box 2 none" "ws2d_box 4 none" "rand0 2 none" "rand1 4 none" "rand2 2 none" "rand3 4 none"; do
  CEL_COPY=tma CEL_NO_GROW=1 timeout 120 python tests/tools/tma_debug.py $c 2>&1 | tail -2
done
unset CUDA_LAUNCH_BLOCKING CEL_EXEC_THREAD
for v in 0 1; do
  CEL_NO_VMM=$v timeout 600 python bench.py --steps 200 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_vmm$v.json 2> gpurun_out/bench_vmm$v.err
  echo "CEL_NO_VMM=$v rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/bench_vmm$v.json'))
print(d['value'], d['roofline']['frac'], d['roofline']['kernel_share_of_step'])
for k,v in d['copy'].items(): print(' ', k, v.get('GBps_hbm_rw'), v.get('frac_hbm'), v.get('us_per_copy'), v.get('bytes_ok'), v.get('kernel'))"
done
