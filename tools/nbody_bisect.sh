port=29850
for f in 0 1; do for n in 2 4; do
  port=$((port+1))
  CEL_NO_FILTER=$f timeout 90 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $port bench_config.py --workload nbody --fast-math --gpus $n --steps 2 > gpurun_out/nb_$f_$n.log 2>&1
  echo "nofilter=$f n=$n rc=$? $(grep '^{' gpurun_out/nb_$f_$n.log | head -1 | cut -c1-120)"
done; done
