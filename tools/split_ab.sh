# shell/interior split on / off at N GPUs
N=${1:-4}
port=29890
for ns in 0 1; do
  port=$((port+1))
  CEL_NO_SPLIT=$ns timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port $port bench.py --gpus $N --steps 4000 --warmup 20 --no-e2e 2>/dev/null | grep "^{" > gpurun_out/sab_$ns.json
  python -c "import json; d=json.load(open('gpurun_out/sab_$ns.json')); print('N=$N nosplit=$ns %.1f steps/s share %.3f' % (d['value'], d['roofline']['kernel_share_of_step']))"
done
