# round 2, 2-GPU call 12: fused halo v3 (boundary strips first) -- parity, A/B of the two halves
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
export OMP_NUM_THREADS=1
CEL_FUSE_HALO=1 timeout 300 $TR --master-port 29601 tests/mp_check.py --execute 1 --quick --only wavesim > gpurun_out/mp_halo_wave.log 2>&1
echo "mp_check wavesim fused rc=$?"; tail -3 gpurun_out/mp_halo_wave.log
run() {  # fuse mode tag
  CEL_FUSE_HALO=$1 CEL_HALO_MODE=$2 timeout 300 $TR --master-port 29620 bench.py --gpus 2 --steps 1000 --warmup 20 --no-e2e > gpurun_out/bench_n2_$3.json 2> gpurun_out/bench_n2_$3.err
  echo "bench N=2 fuse=$1 mode=$2 rc=$?"; tail -1 gpurun_out/bench_n2_$3.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['roofline']['kernel_share_of_step'], d['clocks']['reasons'], d.get('gpu_launches'))"
}
run 0 3 off; run 1 3 m3; run 1 1 m1; run 1 2 m2; run 0 3 off2; run 1 3 m3b
CEL_FUSE_HALO=1 timeout 300 $TR --master-port 29630 tools/trace_wavesim.py > gpurun_out/trace_fused.log 2>&1; echo "trace rc=$?"; tail -16 gpurun_out/trace_fused.log
