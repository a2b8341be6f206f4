# round 2, 4-GPU call 46: Jacobi with programmatic dependent launch -- A/B at 1 and 4 GPUs, parity
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
export OMP_NUM_THREADS=1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
for P in 1 0 1 0; do
  CEL_PDL=$P CEL_BENCH_NOPROF=1 timeout 600 $TR --master-port 29931 bench_config.py --workload jacobi3d --gpus 4 > gpurun_out/j4.json 2> gpurun_out/j4.err
  echo "jacobi 4p pdl=$P rc=$?"; tail -1 gpurun_out/j4.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1))"
  CEL_PDL=$P CEL_BENCH_NOPROF=1 timeout 300 python bench_config.py --workload jacobi3d --gpus 1 > gpurun_out/j1.json 2> gpurun_out/j1.err
  echo "jacobi 1 GPU pdl=$P rc=$?"; tail -1 gpurun_out/j1.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1))"
done
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "jacobi" --timeout 400 --timeout-method thread > gpurun_out/pytest_j.log 2>&1
echo "jacobi parity rc=$?"; tail -2 gpurun_out/pytest_j.log
timeout 600 $TR --master-port 29604 tests/mp_check.py --execute 1 --quick --only jacobi3d > gpurun_out/mp_j.log 2>&1
echo "mp_check jacobi rc=$?"; grep -E "FAIL|MP_CHECK" gpurun_out/mp_j.log | tail -2
