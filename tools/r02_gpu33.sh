# round 2, GPU call 33: the 4096-row chunk kernel of the 4-GPU line on one B200 -- event timing of both variants, ncu --set full of the chosen one
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
for O in 12 16; do CEL_WAVE_OCC=$O timeout 300 python tools/wave_strip.py 4096 | tail -1; done
timeout 300 python tools/wave_strip.py 4096 | tail -1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:wave5_vec -s 30 -c 1 -o gpurun_out/r02_wave5_4096 python tools/wave_strip.py 4096 > gpurun_out/ncu_4096.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/ncu_4096.log
ncu -i gpurun_out/r02_wave5_4096.ncu-rep --page details --csv > gpurun_out/r02_wave5_4096_details.csv 2>/dev/null
grep -E '"Duration"|"DRAM Throughput"|"Memory Throughput"|dram__bytes|"Achieved Occupancy"|"Registers Per Thread"|"Waves Per SM"' gpurun_out/r02_wave5_4096_details.csv | head -12
ncu -i gpurun_out/r02_wave5_4096.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]; v=r[2] if len(r)>2 else r[1]
for k in ('Kernel Name','gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','launch__registers_per_thread','sm__warps_active.avg.pct_of_peak_sustained_active','launch__waves_per_multiprocessor'):
    if k in h: print(k, v[h.index(k)])
"
