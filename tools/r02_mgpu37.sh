# round 2, 4-GPU call 37: fused halo restricted to row bands -- 2-D WaveSim back on the shell path; parity
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
export OMP_NUM_THREADS=1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 600 $TR --master-port 29604 tests/mp_check.py --execute 1 --quick > gpurun_out/mp_q4.log 2>&1
echo "mp_check quick N=4 rc=$?"; grep -E "wavesim|FAIL|MP_CHECK" gpurun_out/mp_q4.log | tail -6
for F in 1 0; do
  CEL_FUSE_HALO=$F timeout 300 $TR --master-port 2993$F bench_config.py --workload wavesim --gpus 4 --split 2d --mapper neighborhood_axes > gpurun_out/w2d_$F.json 2> gpurun_out/w2d_$F.err
  echo "wavesim 2d 4p fuse=$F rc=$?"; tail -1 gpurun_out/w2d_$F.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step']*1e3,1))"
done
timeout 300 $TR --master-port 29939 bench.py --gpus 4 --steps 1000 --warmup 20 --no-e2e > gpurun_out/b4.json 2> gpurun_out/b4.err
echo "bench N=4 rc=$?"; tail -1 gpurun_out/b4.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['kernel'], d['halo_fused_per_step'])"
