# round 2, 4-GPU call 38: 2-D WaveSim at 4 processes -- which change moved it from 6511 (earlier) to ~4400?
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
export OMP_NUM_THREADS=1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
run() { env $1 timeout 300 $TR --master-port 29930 bench_config.py --workload wavesim --gpus 4 --split 2d --mapper neighborhood_axes > gpurun_out/w2d.json 2> gpurun_out/w2d.err
  echo "$1 rc=$?"; tail -1 gpurun_out/w2d.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step']*1e3,1), d.get('profile_ms'))"; }
run CEL_X=0; run CEL_WAVE_OCC=12; run CEL_SCHED_MEMO=0; run CEL_BENCH_NOPROF=1; run "CEL_WAVE_OCC=12 CEL_BENCH_NOPROF=1"
