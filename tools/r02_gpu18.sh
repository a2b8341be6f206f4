# round 2, GPU call 18: wave5 cache-hint variants (strip 8)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
for rows in 16384 4096; do for v in 0 1 2 0 1 2; do CEL_WAVE_VAR=$v timeout 120 python tools/wave_strip.py $rows | sed "s/^/var $v /"; done; done
