#!/bin/bash
# Multi-GPU runs of the other configs (bench_config.py); one JSON line per run.
NG=${1:-4}
for wl in jacobi3d nbody; do
  for n in 1 2 4; do
    [ $n -gt $NG ] && continue
    if [ $n -eq 1 ]; then
      timeout 300 python bench_config.py --workload $wl --gpus 1 $EXTRA
    else
      timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2960$n bench_config.py --workload $wl --gpus $n $EXTRA 2>&1 | grep '^{'
    fi
  done
done
for la in auto none; do
  for n in 1 4; do
    [ $n -gt $NG ] && continue
    if [ $n -eq 1 ]; then
      timeout 300 python bench_config.py --workload rsim --gpus 1 --lookahead $la
    else
      timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2961$n bench_config.py --workload rsim --gpus $n --lookahead $la 2>&1 | grep '^{'
    fi
  done
done
EXTRA=--fast-math
for n in 1 4; do
  [ $n -gt $NG ] && continue
  if [ $n -eq 1 ]; then timeout 300 python bench_config.py --workload nbody --gpus 1 --fast-math
  else timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2962$n bench_config.py --workload nbody --gpus $n --fast-math 2>&1 | grep '^{'; fi
done
