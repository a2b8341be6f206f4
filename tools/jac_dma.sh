port=29940
for v in 0 1; do
  port=$((port+1))
  CEL_PEER_DMA=$v timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port $port bench_config.py --workload jacobi3d --gpus 4 2>/dev/null | grep "^{" | head -1 > gpurun_out/jdma_$v.json
  python -c "import json; d=json.load(open('gpurun_out/jdma_$v.json')); print('jacobi N=4 peer_dma=$v %.1f steps/s' % d['value'])"
  port=$((port+1))
  CEL_PEER_DMA=$v timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port $port bench.py --gpus 4 --steps 4000 --warmup 20 --no-e2e --no-cpu-baseline 2>/dev/null | grep "^{" > gpurun_out/wdma_$v.json
  python -c "import json; d=json.load(open('gpurun_out/wdma_$v.json')); print('wavesim N=4 peer_dma=$v %.1f steps/s' % d['value'])"
done
