# round 2, 4-GPU call 27: RSim fused -- is it the kernel or the wait chain? (in-kernel waits off / fusion off, profiled)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
export OMP_NUM_THREADS=1
show() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step']*1e3,1), {k: (round(v['ms'],2), v['launches']) for k,v in d['profile_ms'].items()})"; }
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
CEL_HALO_MODE=1 timeout 300 $TR --master-port 29911 bench_config.py --workload rsim --gpus 4 > gpurun_out/r4_m1.json 2> gpurun_out/r4_m1.err; echo "fused, stream waits, prof rc=$?"; show gpurun_out/r4_m1.json
CEL_FUSE_HALO=0 timeout 300 $TR --master-port 29912 bench_config.py --workload rsim --gpus 4 > gpurun_out/r4_m0.json 2> gpurun_out/r4_m0.err; echo "unfused prof rc=$?"; show gpurun_out/r4_m0.json
CEL_PDL=0 timeout 300 $TR --master-port 29913 bench_config.py --workload rsim --gpus 4 > gpurun_out/r4_np.json 2> gpurun_out/r4_np.err; echo "fused, no PDL, prof rc=$?"; show gpurun_out/r4_np.json
CEL_BENCH_NOPROF=1 CEL_HALO_MODE=1 timeout 300 $TR --master-port 29914 bench_config.py --workload rsim --gpus 4 > gpurun_out/r4_m1n.json 2> gpurun_out/r4_m1n.err; echo "fused, stream waits, noprof rc=$?"; show gpurun_out/r4_m1n.json
