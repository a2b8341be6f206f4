# round 2, 4-GPU call 6: suite with multi-process P2P only for large sets and no fusion across processes
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 --timeout-method thread > gpurun_out/pytest.log 2>&1
echo "pytest all rc=$?"; tail -3 gpurun_out/pytest.log; grep -E "^E |^FAILED" gpurun_out/pytest.log | head -20
j() { python -c "
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
keys=('value','ms_per_step','gen_us_per_step','coll_groups','coll_p2p','coll_fused','coll_allgathers','GBps_received_per_device')
print({k: d.get(k) for k in keys}, {k: v for k, v in d.get('profile_ms', {}).items() if k in ('coll','rsim_row','nbody_step')})" $1; }
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29661 bench_config.py --workload rsim --gpus 4 > gpurun_out/r4.json 2> gpurun_out/r4.err
echo "rsim 4 processes rc=$?"; j gpurun_out/r4.json
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29662 bench_config.py --workload gather --gpus 4 > gpurun_out/g4.json 2> gpurun_out/g4.err
echo "gather 4 processes rc=$?"; j gpurun_out/g4.json
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29663 bench_config.py --workload nbody --gpus 4 --fast-math > gpurun_out/n4.json 2> gpurun_out/n4.err
echo "nbody fast 4 processes rc=$?"; j gpurun_out/n4.json
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29664 bench_config.py --workload jacobi3d --gpus 4 > gpurun_out/j4.json 2> gpurun_out/j4.err
echo "jacobi 4 processes rc=$?"; tail -c 400 gpurun_out/j4.json
