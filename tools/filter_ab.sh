# rank filter on / off: WaveSim bench host cost and RSim rows/s at 4 GPUs
port=29870
for f in 0 1; do
  port=$((port+1))
  CEL_NO_FILTER=$f timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port $port bench.py --gpus 4 --steps 4000 --warmup 20 --no-e2e 2>/dev/null | grep "^{" > gpurun_out/fab_$f.json
  python -c "import json; d=json.load(open('gpurun_out/fab_$f.json')); print('nofilter=$f wavesim %.1f host %.1f us/step' % (d['value'], d['host_submit_us_per_step']), {k: round(v, 1) for k, v in d['host_us_per_step_by_part'].items()})"
  port=$((port+1))
  CEL_NO_FILTER=$f timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port $port bench_config.py --workload rsim --gpus 4 2>/dev/null | grep "^{" | head -1 > gpurun_out/fabr_$f.json
  python -c "import json; d=json.load(open('gpurun_out/fabr_$f.json')); print('nofilter=$f rsim %.1f rows/s gen %.1f us/row' % (d['value'], d['gen_us_per_step']))"
done
