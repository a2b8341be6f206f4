# round 2, 4-GPU call 30: wave5 at 16 CTAs/SM (32 registers) vs 12 (40) -- N=1 and N=4 fused
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
export OMP_NUM_THREADS=1
for O in 12 16 12 16; do
  CEL_WAVE_OCC=$O timeout 300 python bench.py --steps 1000 --warmup 20 --no-e2e --no-cpu-baseline --no-copy > gpurun_out/b1_$O.json 2> gpurun_out/b1_$O.err
  echo "N=1 occ=$O rc=$?"; tail -1 gpurun_out/b1_$O.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
for O in 12 16 16 12; do
  for S in 0 8; do
    CEL_WAVE_OCC=$O CEL_WAVE_STRIP=$S timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29640 bench.py --gpus 4 --steps 1000 --warmup 20 --no-e2e > gpurun_out/b4_$O.json 2> gpurun_out/b4_$O.err
    echo "N=4 occ=$O strip=$S rc=$?"; tail -1 gpurun_out/b4_$O.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['roofline']['frac'],3), round(d['roofline']['kernel_share_of_step'],3), d['clocks']['reasons'])"
  done
done
