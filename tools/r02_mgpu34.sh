# round 2, 4-GPU call 34: wave5 variant A/B at N=2 and N=3 (fused halo): 12 vs 16 CTAs/SM
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
export OMP_NUM_THREADS=1
for N in 2 3; do
for O in 12 16 12 16; do
  CEL_WAVE_OCC=$O timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29640 bench.py --gpus $N --steps 1000 --warmup 20 --no-e2e > gpurun_out/bx.json 2> gpurun_out/bx.err
  echo "N=$N occ=$O rc=$?"; tail -1 gpurun_out/bx.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['roofline']['frac'],3), round(d['roofline']['kernel_share_of_step'],3), d['clocks']['reasons'])"
done
done
