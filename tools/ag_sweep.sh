# N-body 2^20 fast-math at N GPUs: the all-gather set as ncclAllGather / grouped ncclBroadcast / peer pushes
N=${1:-4}
run() {   # $1 collective, $2 CEL_COLL_AG
  CEL_COLL_AG=$2 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port 29${N}$1$2 bench_config.py --workload nbody --fast-math --gpus $N --steps 6 --collective $1 \
    > gpurun_out/ag_${N}_$1$2.log 2>&1
  grep "^{" gpurun_out/ag_${N}_$1$2.log | head -1 > gpurun_out/ag_${N}_$1$2.json
  python -c "import json; d=json.load(open('gpurun_out/ag_${N}_$1$2.json')); print('N=$N collective=$1 allgather=$2 %.3f steps/s ag=%d bc=%d coll_ms=%s' % (d['value'], d['coll_allgathers'], d['coll_groups'], d['profile_ms'].get('coll', {}).get('ms')))"
}
run 1 1
run 1 0
run 0 1
