# Round-end measurement batch (4 GPUs): bench N=1 (+ncu launch list), N=2, N=4; suite; configs
set -x
mkdir -p gpurun_out/final
timeout 400 python bench.py > gpurun_out/final/bench_n1.json 2> gpurun_out/final/bench_n1.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/final/launches_n1.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e \
  > gpurun_out/final/ncu_n1.log 2>&1
for N in 2 4; do
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port 2950$N bench.py --gpus $N --steps 4000 --warmup 20 > gpurun_out/final/bench_n$N.log 2>&1
  grep "^{" gpurun_out/final/bench_n$N.log > gpurun_out/final/bench_n$N.json
done
timeout 600 python bench_suite.py > gpurun_out/final/suite.log 2>&1
port=29600
for w in jacobi3d nbody rsim; do for N in 1 2 4; do
  port=$((port+1))
  if [ $N = 1 ]; then
    timeout 300 python bench_config.py --workload $w --gpus 1 2>/dev/null | grep "^{" | head -1 >> gpurun_out/final/configs.jsonl
  else
    timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $port \
      bench_config.py --workload $w --gpus $N 2>/dev/null | grep "^{" | head -1 >> gpurun_out/final/configs.jsonl
  fi
done; done
port=29700
for N in 1 4; do
  port=$((port+1))
  if [ $N = 1 ]; then
    timeout 300 python bench_config.py --workload nbody --fast-math --gpus 1 2>/dev/null | grep "^{" | head -1 >> gpurun_out/final/configs.jsonl
    timeout 300 python bench_config.py --workload rsim --lookahead none --gpus 1 2>/dev/null | grep "^{" | head -1 >> gpurun_out/final/configs.jsonl
  else
    timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $port \
      bench_config.py --workload nbody --fast-math --gpus $N 2>/dev/null | grep "^{" | head -1 >> gpurun_out/final/configs.jsonl
  fi
done
