# round 2, 4-GPU call 3: P2P gather kernels (default) vs NCCL / pushes / multicast; RSim and gather in 1 and 4 processes
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q --timeout 300 --timeout-method thread -k "multicast or physical_multi or collective_vs or distinct_gpus or multiprocess_gpu" > gpurun_out/pytest_mgpu.log 2>&1
echo "pytest mgpu rc=$?"; grep -E "^E |passed|failed" gpurun_out/pytest_mgpu.log | head
j() { python -c "
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
keys=('value','ms_per_step','gen_us_per_step','exec_us_per_step','coll_groups','coll_p2p','coll_multicast','coll_allgathers','GBps_received_per_device')
print({k: d.get(k) for k in keys}, {k: v for k, v in d.get('profile_ms', {}).items() if k in ('coll','rsim_row','copy_peer')})" $1; }
for cfg in "P2P" "NCCL:CEL_COLL_P2P=0" "MC:CEL_COLL_MC=1" "PUSH:--collective 0"; do
  name=${cfg%%:*}; arg=${cfg#*:}; envs=""; flags=""
  case "$arg" in CEL_*) envs=$arg;; --*) flags=$arg;; esac
  [ "$name" = "P2P" ] && envs="" && flags=""
  env $envs timeout 300 python bench_config.py --workload gather --gpus 4 $flags > gpurun_out/g1_$name.json 2> gpurun_out/g1_$name.err
  echo "gather 1 process $name rc=$?"; j gpurun_out/g1_$name.json
  env $envs timeout 300 python bench_config.py --workload rsim --gpus 4 $flags > gpurun_out/r1_$name.json 2> gpurun_out/r1_$name.err
  echo "rsim 1 process $name rc=$?"; j gpurun_out/r1_$name.json
done
for cfg in "P2P" "NCCL:CEL_COLL_P2P=0"; do
  name=${cfg%%:*}; envs=""; [ "$name" != "P2P" ] && envs=${cfg#*:}
  env $envs timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29621 bench_config.py --workload gather --gpus 4 > gpurun_out/g4_$name.json 2> gpurun_out/g4_$name.err
  echo "gather 4 processes $name rc=$?"; j gpurun_out/g4_$name.json
  env $envs timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29622 bench_config.py --workload rsim --gpus 4 > gpurun_out/r4_$name.json 2> gpurun_out/r4_$name.err
  echo "rsim 4 processes $name rc=$?"; j gpurun_out/r4_$name.json
  env $envs timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29623 bench_config.py --workload rsim --gpus 2 > gpurun_out/r2_$name.json 2> gpurun_out/r2_$name.err
  echo "rsim 2 processes $name rc=$?"; j gpurun_out/r2_$name.json
done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29624 bench_config.py --workload nbody --gpus 4 --fast-math > gpurun_out/n4.json 2> gpurun_out/n4.err
echo "nbody fast 4 processes P2P rc=$?"; j gpurun_out/n4.json
