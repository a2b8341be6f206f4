mkdir -p gpurun_out/final4
port=29600
for w in jacobi3d nbody rsim; do for N in 2 4; do
  port=$((port+1))
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $port \
    bench_config.py --workload $w --gpus $N 2>/dev/null | grep "^{" | head -1 >> gpurun_out/final4/configs.jsonl
done; done
port=29700
for N in 2 4; do
  port=$((port+1))
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $port \
    bench_config.py --workload nbody --fast-math --gpus $N 2>/dev/null | grep "^{" | head -1 >> gpurun_out/final4/configs.jsonl
done
python -c "
import json
for l in open('gpurun_out/final4/configs.jsonl'):
    d = json.loads(l); print(d['workload'], d['n_gpus'], round(d['value'], 2), d['unit'], d.get('roofline', {}).get('fast_math', ''))
"
