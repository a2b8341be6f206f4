# round 2, 4-GPU call 13: fused halo at 4 GPUs -- multi-process tests, A/B at N=4
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
export OMP_NUM_THREADS=1
timeout 900 python -m pytest tests/test_multiprocess.py -m gpu -q --timeout 400 --timeout-method thread > gpurun_out/pytest_mp4.log 2>&1
echo "pytest multiprocess (4 GPUs) rc=$?"; tail -3 gpurun_out/pytest_mp4.log; grep -E "^E |FAILED" gpurun_out/pytest_mp4.log | head
run() {  # N fuse tag
  TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1"
  CEL_FUSE_HALO=$2 timeout 300 $TR --master-port 29640 bench.py --gpus $1 --steps 1000 --warmup 20 --no-e2e > gpurun_out/bench_n$1_$3.json 2> gpurun_out/bench_n$1_$3.err
  echo "bench N=$1 fuse=$2 rc=$?"; tail -1 gpurun_out/bench_n$1_$3.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['roofline']['kernel_share_of_step'], d['clocks']['reasons'], d.get('gpu_launches'), d.get('halo_fused_per_step'))"
}
run 4 0 off; run 4 1 on; run 4 0 off2; run 4 1 on2; run 2 1 on; run 3 1 on; run 3 0 off
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
CEL_FUSE_HALO=1 timeout 300 $TR --master-port 29650 tools/trace_wavesim.py > gpurun_out/trace_fused4.log 2>&1; echo "trace rc=$?"; tail -8 gpurun_out/trace_fused4.log
