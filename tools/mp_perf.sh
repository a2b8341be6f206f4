# multi-process parity + WaveSim / config benches at 4 GPUs (host-cost check)
timeout 600 python -m pytest tests/test_multiprocess.py -x -q -m gpu 2>&1 | tail -2
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29814 \
  bench.py --gpus 4 --steps 4000 --warmup 20 --no-e2e 2>/dev/null | grep "^{" > gpurun_out/bn4c.json
python -c "import json; d=json.load(open('gpurun_out/bn4c.json')); print('wavesim', d['value'], d['host_submit_us_per_step'], d['host_us_per_step_by_part'])"
port=29830
for p in jacobi3d nbody rsim; do
  port=$((port+1))
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $port \
    bench_config.py --workload $p --gpus 4 2>/dev/null | grep "^{" | head -1 | cut -c1-260
done
