# round 2, 4-GPU call 42: final validation of the committed tree -- suite on 4 GPUs, smoke, bench N=1 / N=4
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
export OMP_NUM_THREADS=1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 400 --timeout-method thread > gpurun_out/pytest4.log 2>&1
echo "pytest all (4 GPUs) rc=$?"; tail -2 gpurun_out/pytest4.log; grep -E "^E |^FAILED" gpurun_out/pytest4.log | head -20
CUDA_VISIBLE_DEVICES=0 timeout 1500 python -m pytest tests -m gpu -q --timeout 400 --timeout-method thread > gpurun_out/pytest1.log 2>&1
echo "pytest one GPU rc=$?"; tail -2 gpurun_out/pytest1.log
timeout 900 python bench.py > gpurun_out/final_n1_default.json 2> gpurun_out/final_n1_default.err
echo "bench default rc=$?"; tail -1 gpurun_out/final_n1_default.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['e2e']['value'], d['gpu_launches'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29904 bench.py --gpus 4 --steps 1000 --warmup 20 > gpurun_out/final_n4.json 2> gpurun_out/final_n4.err
echo "bench N=4 rc=$?"; tail -1 gpurun_out/final_n4.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['kernel'], d['roofline']['frac'], d['e2e']['value'])"
