# round 2, 4-GPU call 36: fused halo with the 2-D split (tiles: row bands fused, column strips as copies) -- parity, A/B
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
export OMP_NUM_THREADS=1
for N in 4 2; do
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
timeout 600 $TR --master-port 2960$N tests/mp_check.py --execute 1 --quick > gpurun_out/mp_q$N.log 2>&1
echo "mp_check quick N=$N rc=$?"; grep -E "wavesim2d|FAIL|MP_CHECK|halo" gpurun_out/mp_q$N.log | tail -6
done
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
for F in 1 0; do
  CEL_FUSE_HALO=$F timeout 300 $TR --master-port 2993$F bench_config.py --workload wavesim --gpus 4 --split 2d --mapper neighborhood_axes > gpurun_out/w2d_$F.json 2> gpurun_out/w2d_$F.err
  echo "wavesim 2d 4p fuse=$F rc=$?"; tail -1 gpurun_out/w2d_$F.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step']*1e3,1))"
done
