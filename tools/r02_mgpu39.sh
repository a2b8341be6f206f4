# round 2, 4-GPU call 39: narrow-row peer pushes on the copy kernel instead of 2-D DMA -- 2-D WaveSim, Jacobi, parity
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
export OMP_NUM_THREADS=1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
for O in 0 12; do
  CEL_WAVE_OCC=$O CEL_BENCH_NOPROF=1 timeout 300 $TR --master-port 29930 bench_config.py --workload wavesim --gpus 4 --split 2d --mapper neighborhood_axes > gpurun_out/w2d.json 2> gpurun_out/w2d.err
  echo "wavesim 2d occ=$O rc=$?"; tail -1 gpurun_out/w2d.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step']*1e3,1))"
done
timeout 300 $TR --master-port 29931 bench_config.py --workload jacobi3d --gpus 4 > gpurun_out/j4.json 2> gpurun_out/j4.err
echo "jacobi 4p rc=$?"; tail -1 gpurun_out/j4.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['ms_per_step']*1e3,1))"
timeout 600 $TR --master-port 29604 tests/mp_check.py --execute 1 --quick > gpurun_out/mp_q4.log 2>&1
echo "mp_check quick N=4 rc=$?"; grep -E "FAIL|MP_CHECK" gpurun_out/mp_q4.log | tail -2
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 400 --timeout-method thread > gpurun_out/pytest_p.log 2>&1
echo "parity rc=$?"; tail -2 gpurun_out/pytest_p.log
