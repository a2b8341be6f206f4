# round 2, 4-GPU call 2: multicast on VMM allocations; gather / RSim / N-body A/B; ncu NVLink counters
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 300 --timeout-method thread -k "multicast" > gpurun_out/pytest_mc.log 2>&1
echo "pytest multicast rc=$?"; grep -E "^E |passed|failed" gpurun_out/pytest_mc.log | head
for cfg in "0 0" "1 0" "1 1"; do
  set -- $cfg
  CEL_COLL_MC=$2 NCCL_DEBUG=WARN timeout 300 python -X faulthandler bench_config.py --workload gather --gpus 4 --collective $1 > gpurun_out/gather_c$1_m$2.json 2> gpurun_out/gather_c$1_m$2.err
  echo "gather 1 process collective=$1 mc=$2 rc=$?"; cat gpurun_out/gather_c$1_m$2.json; tail -3 gpurun_out/gather_c$1_m$2.err
done
for mc in 0 1; do
  CEL_COLL_MC=$mc timeout 300 python -X faulthandler bench_config.py --workload rsim --gpus 4 > gpurun_out/rsim_m$mc.json 2> gpurun_out/rsim_m$mc.err
  echo "rsim 1 process mc=$mc rc=$?"; cat gpurun_out/rsim_m$mc.json; tail -3 gpurun_out/rsim_m$mc.err
done
for mc in 0 1; do
  CEL_COLL_MC=$mc timeout 300 python -X faulthandler bench_config.py --workload nbody --gpus 4 --fast-math > gpurun_out/nbody_m$mc.json 2> gpurun_out/nbody_m$mc.err
  echo "nbody fast 1 process mc=$mc rc=$?"; cat gpurun_out/nbody_m$mc.json; tail -3 gpurun_out/nbody_m$mc.err
done
timeout 120 python tools/peer_case.py push 2 256 && timeout 120 python tools/peer_case.py mc 4 16 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum \
  --clock-control none -k regex:"copy_kernel|mc_gather" --csv --log-file gpurun_out/ncu_nvlink_push.csv python tools/peer_case.py push 2 256 > gpurun_out/ncu_push.log 2>&1
echo "ncu push rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum \
  --clock-control none -k regex:"copy_kernel|mc_gather" --csv --log-file gpurun_out/ncu_nvlink_mc.csv python tools/peer_case.py mc 4 16 > gpurun_out/ncu_mc.log 2>&1
echo "ncu mc rc=$?"
