# round 2, 4-GPU call 16: fused halo + step chain (per-strip counters instead of griddepcontrol.wait) -- parity, A/B
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
export OMP_NUM_THREADS=1
for N in 2 4; do
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
CEL_FUSE_HALO=1 timeout 300 $TR --master-port 2960$N tests/mp_check.py --execute 1 --quick --only wavesim > gpurun_out/mp_halo_wave$N.log 2>&1
echo "mp_check wavesim fused N=$N rc=$?"; grep -E "halo|MP_CHECK" gpurun_out/mp_halo_wave$N.log | tail -3
done
run() {  # N fuse chain tag
  TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1"
  CEL_FUSE_HALO=$2 CEL_HALO_CHAIN=$3 timeout 300 $TR --master-port 29640 bench.py --gpus $1 --steps 1000 --warmup 20 --no-e2e > gpurun_out/bench_n$1_$4.json 2> gpurun_out/bench_n$1_$4.err
  echo "bench N=$1 fuse=$2 chain=$3 rc=$?"; tail -1 gpurun_out/bench_n$1_$4.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['roofline']['kernel_share_of_step'], d['clocks']['reasons'], d.get('gpu_launches'), d.get('halo_fused_per_step'), d.get('halo_chained_per_step'))"
}
run 4 1 1 chain; run 4 1 0 nochain; run 4 0 1 off; run 4 1 1 chainb; run 2 1 1 chain; run 2 1 0 nochain; run 3 1 1 chain
tail -3 gpurun_out/bench_n4_chain.err
