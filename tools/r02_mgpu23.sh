# round 2, 4-GPU call 23: fused RSim rows (flag mode) after the in-wait id fix -- full mp_check at 2 / 4, A/B
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
export OMP_NUM_THREADS=1
for N in 2 4; do
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
timeout 600 $TR --master-port 2960$N tests/mp_check.py --execute 1 > gpurun_out/mp_all$N.log 2>&1
echo "mp_check all N=$N rc=$?"; grep -E "FAIL|MP_CHECK|halo" gpurun_out/mp_all$N.log | tail -8
done
show() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step']*1e3,1), round(d['gen_us_per_step'],1), {k: round(v,1) for k,v in d['exec_us_per_step'].items()}, {k: round(v,2) for k,v in d['per_step'].items()})"; }
for F in 1 0; do
  CEL_FUSE_HALO=$F CEL_BENCH_NOPROF=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2991$F bench_config.py --workload rsim --gpus 4 > gpurun_out/r4_f$F.json 2> gpurun_out/r4_f$F.err
  echo "rsim 4 processes fuse=$F rc=$?"; show gpurun_out/r4_f$F.json
done
CEL_BENCH_NOPROF=1 timeout 300 python bench_config.py --workload rsim --gpus 1 > gpurun_out/r1g.json 2> gpurun_out/r1g.err; echo "rsim 1 GPU rc=$?"; show gpurun_out/r1g.json
