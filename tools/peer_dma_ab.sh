# halo pushes as SM copy kernels (default) vs copy-engine DMA (CEL_PEER_DMA=1)
N=${1:-4}
port=29930
for v in 0 1; do
  port=$((port+1))
  CEL_PEER_DMA=$v timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port $port bench.py --gpus $N --steps 4000 --warmup 20 --no-e2e 2>/dev/null | grep "^{" > gpurun_out/pdma_$v.json
  python -c "import json; d=json.load(open('gpurun_out/pdma_$v.json')); print('N=$N peer_dma=$v %.1f steps/s share %.3f' % (d['value'], d['roofline']['kernel_share_of_step']), d['profile_ms'].get('copy_peer'))"
done
