# round 2, 4-GPU call 1: multi-GPU tests, WaveSim scaling, gather / RSim / N-body A/B (multicast, NCCL, pushes)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
nvidia-smi topo -m > gpurun_out/topo.txt 2>&1; head -8 gpurun_out/topo.txt
timeout 300 python tools/peer_peak.py > gpurun_out/peer_peak.json 2>&1; cat gpurun_out/peer_peak.json
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -k "multicast or physical_multi or collective_vs or distinct_gpus or multiprocess_gpu or direct" > gpurun_out/pytest_mgpu.log 2>&1
echo "pytest mgpu rc=$?"; tail -25 gpurun_out/pytest_mgpu.log
timeout 600 python bench.py --gpus 1 --steps 1000 --warmup 20 --no-e2e --no-cpu-baseline --no-copy > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err
echo "bench N=1 rc=$?"; python -c "import json; d=json.loads(open('gpurun_out/bench_n1.json').read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'], d['roofline']['kernel_share_of_step'], d['clocks'])"
for N in 2 4; do
  for pin in 1 0; do
    CEL_PIN=$pin timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 295$N$pin bench.py --gpus $N --steps 1000 --warmup 20 --no-e2e > gpurun_out/bench_n${N}_pin$pin.json 2> gpurun_out/bench_n${N}_pin$pin.err
    echo "bench N=$N pin=$pin rc=$?"; python -c "import json; d=json.loads(open('gpurun_out/bench_n${N}_pin$pin.json').read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'], d['roofline']['kernel_share_of_step'], d['clocks'], d['host_submit_us_per_step'])"
  done
done
for cfg in "--collective 0" "--collective 1" "--collective 1 MC"; do
  mc=0; case "$cfg" in *MC*) mc=1;; esac; c=${cfg% MC}
  CEL_COLL_MC=$mc timeout 300 python bench_config.py --workload gather --gpus 4 $c > gpurun_out/gather.json 2> gpurun_out/gather.err
  echo "gather 4 GPUs 1 process $cfg rc=$?"; cat gpurun_out/gather.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k: d[k] for k in ('value','ms_per_step','GBps_received_per_device','frac_nvlink_measured_ref','coll_groups','coll_multicast','coll_allgathers')})"
done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29611 bench_config.py --workload gather --gpus 4 > gpurun_out/gather_mp.json 2> gpurun_out/gather_mp.err
echo "gather 4 processes NCCL rc=$?"; tail -1 gpurun_out/gather_mp.json
for cfg in "0" "1"; do
  CEL_COLL_MC=$cfg timeout 300 python bench_config.py --workload rsim --gpus 4 > gpurun_out/rsim.json 2> gpurun_out/rsim.err
  echo "rsim 4 GPUs 1 process MC=$cfg rc=$?"; cat gpurun_out/rsim.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k: d.get(k) for k in ('value','ms_per_step','host_ms_per_step','gen_us_per_step','coll_groups')}, d['profile_ms'])"
done
timeout 300 python bench_config.py --workload rsim --gpus 1 > gpurun_out/rsim1.json 2> gpurun_out/rsim1.err; echo "rsim 1 GPU"; cat gpurun_out/rsim1.json
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29612 bench_config.py --workload rsim --gpus 4 > gpurun_out/rsim_mp.json 2> gpurun_out/rsim_mp.err
echo "rsim 4 processes rc=$?"; tail -1 gpurun_out/rsim_mp.json
for mc in 0 1; do
  CEL_COLL_MC=$mc timeout 300 python bench_config.py --workload nbody --gpus 4 --fast-math > gpurun_out/nbody.json 2> gpurun_out/nbody.err
  echo "nbody fast 4 GPUs 1 process MC=$mc rc=$?"; cat gpurun_out/nbody.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k: d.get(k) for k in ('value','ms_per_step','coll_groups')}, d['profile_ms'].get('coll'))"
done
CEL_DIRECT_SENDS=1 timeout 600 python -m pytest tests/test_gpu_cluster.py -m gpu -q --timeout 180 --timeout-method thread > gpurun_out/pytest_cluster_direct.log 2>&1
echo "cluster tests with direct sends rc=$?"; tail -3 gpurun_out/pytest_cluster_direct.log
