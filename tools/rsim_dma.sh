port=29950
for v in 1 0; do
  port=$((port+1))
  CEL_PEER_DMA=$v timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port $port bench_config.py --workload rsim --gpus 4 2>/dev/null | grep "^{" | head -1 > gpurun_out/rdma_$v.json
  python -c "import json; d=json.load(open('gpurun_out/rdma_$v.json')); print('rsim N=4 peer_dma=$v %.1f rows/s' % d['value'])"
done
