# WaveSim bench with and without the live per-launch profile (CUDA events around each launch)
N=${1:-4}
for np in "" 1; do
  CEL_BENCH_NOPROF=$np timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
    --master-addr 127.0.0.1 --master-port 298$N${np:-0} bench.py --gpus $N --steps 3000 --warmup 20 \
    --no-cpu-baseline --no-e2e 2>/dev/null | grep "^{" > gpurun_out/prof_${N}_${np:-0}.json
  python -c "import json; d=json.load(open('gpurun_out/prof_${N}_${np:-0}.json')); print('N=$N noprof=${np:-0} value=%.1f ms/step=%.4f' % (d['value'], d['ms_per_step']))"
done
