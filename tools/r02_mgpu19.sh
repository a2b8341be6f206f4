# round 2, 4-GPU call 19: RSim rows fused with their pushes across processes (flag mode) -- parity, A/B
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
export OMP_NUM_THREADS=1
for N in 2 4; do
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
timeout 300 $TR --master-port 2960$N tests/mp_check.py --execute 1 --quick --only rsim > gpurun_out/mp_rsim$N.log 2>&1
echo "mp_check rsim N=$N rc=$?"; grep -E "halo|rsim|MP_CHECK" gpurun_out/mp_rsim$N.log | tail -5
done
show() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step']*1e3,1), round(d['gen_us_per_step'],1), {k: round(v,1) for k,v in d['exec_us_per_step'].items()}, {k: round(v,1) for k,v in d['host_us_per_step'].items()}, {k: round(v,2) for k,v in d['per_step'].items()})"; }
for F in 1 0 1 0; do
  CEL_FUSE_HALO=$F CEL_BENCH_NOPROF=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2991$F bench_config.py --workload rsim --gpus 4 > gpurun_out/r4_f$F.json 2> gpurun_out/r4_f$F.err
  echo "rsim 4 processes fuse=$F rc=$?"; show gpurun_out/r4_f$F.json
done
CEL_BENCH_NOPROF=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29930 bench_config.py --workload rsim --gpus 2 > gpurun_out/r2_f1.json 2> gpurun_out/r2_f1.err
echo "rsim 2 processes fuse=1 rc=$?"; show gpurun_out/r2_f1.json
tail -3 gpurun_out/r4_f1.err
