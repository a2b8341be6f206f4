# round 2, 4-GPU call 43: Jacobi 1024^3 at 4 processes -- where the last 10% goes (profile, DMA off)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
export OMP_NUM_THREADS=1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
show() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['ms_per_step']*1e3,1), {k: (round(v['ms'],2), v['launches']) for k,v in d.get('profile_ms',{}).items()}, {k: round(v,2) for k,v in d.get('per_step',{}).items()})"; }
run() { env $1 timeout 600 $TR --master-port 29931 bench_config.py --workload jacobi3d --gpus 4 > gpurun_out/j.json 2> gpurun_out/j.err; echo "$1 rc=$?"; show gpurun_out/j.json; }
run CEL_X=1; run CEL_PEER_DMA=0; run CEL_BENCH_NOPROF=1
timeout 300 python bench_config.py --workload jacobi3d --gpus 1 > gpurun_out/j1.json 2> gpurun_out/j1.err; echo "1 GPU rc=$?"; show gpurun_out/j1.json
