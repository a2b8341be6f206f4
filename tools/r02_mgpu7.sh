# round 2, 4-GPU call 7: final multi-GPU suite; virtual nodes with device-direct sends vs M1 staging; WaveSim N=2/4
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 --timeout-method thread > gpurun_out/pytest4.log 2>&1
echo "pytest all (4 GPUs) rc=$?"; tail -3 gpurun_out/pytest4.log; grep -E "^E |^FAILED" gpurun_out/pytest4.log | head -20
: > gpurun_out/r02_nodes.jsonl
for cfg in "2 1 wavesim" "4 1 wavesim" "2 2 wavesim" "4 1 nbody" "2 2 nbody"; do
  set -- $cfg
  for ds in 1 0; do
    CEL_DIRECT_SENDS=$ds timeout 600 python bench_nodes.py --nodes $1 --devices-per-node $2 --workload $3 >> gpurun_out/r02_nodes.jsonl 2> gpurun_out/nodes.err
    echo "nodes $cfg direct=$ds rc=$?"; tail -1 gpurun_out/r02_nodes.jsonl | python -c "import json,sys; d=json.loads(sys.stdin.read()); v=d['virtual_nodes']; print(v['steps_per_s'], v['staging_copies_elided_per_step'], v['pull_GBps'], 'single node', d['single_node']['steps_per_s'])"
  done
done
for N in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2970$N bench.py --gpus $N --steps 1000 --warmup 20 --no-e2e > gpurun_out/bench_n$N.json 2> gpurun_out/bench_n$N.err
  echo "bench N=$N rc=$?"; tail -1 gpurun_out/bench_n$N.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['roofline']['kernel_share_of_step'], d['clocks'])"
done
