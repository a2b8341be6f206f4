# WaveSim 16384^2 at 4 GPUs: 1-D vs 2-D split, box vs axis-only neighbourhood
port=29740
for v in "1d neighborhood" "2d neighborhood" "2d neighborhood_axes"; do
  set -- $v
  port=$((port+1))
  timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $port \
    bench_config.py --workload wavesim --gpus 4 --split $1 --mapper $2 2>/dev/null | grep "^{" | head -1 > gpurun_out/ws2d_$1_$2.json
  python -c "import json; d=json.load(open('gpurun_out/ws2d_$1_$2.json')); print('$1 $2 %.1f steps/s, %.1f coherence copies/step' % (d['value'], d['coherence_copies_per_step']))"
done
