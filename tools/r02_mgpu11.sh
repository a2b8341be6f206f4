# round 2, 2-GPU call 11: fused halo kernel v2 (forwarding after the strip, 40 regs) -- parity, A/B; PDL probe
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
export OMP_NUM_THREADS=1
CEL_FUSE_HALO=1 timeout 300 $TR --master-port 29601 tests/mp_check.py --execute 1 --quick --only wavesim > gpurun_out/mp_halo_wave.log 2>&1
echo "mp_check wavesim fused rc=$?"; tail -5 gpurun_out/mp_halo_wave.log
for F in 0 1 0 1; do
  CEL_FUSE_HALO=$F timeout 300 $TR --master-port 2961$F bench.py --gpus 2 --steps 1000 --warmup 20 --no-e2e > gpurun_out/bench_n2_h$F.json 2> gpurun_out/bench_n2_h$F.err
  echo "bench N=2 fuse=$F rc=$?"; tail -1 gpurun_out/bench_n2_h$F.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['roofline']['kernel_share_of_step'], d['clocks']['reasons'], d.get('gpu_launches'))"
done
nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/pdl_probe.cu -o /tmp/pdl_probe && /tmp/pdl_probe
