# round 2, 4-GPU call 25: RSim fused, per-launch profile (kernel time incl. in-kernel waits) at 4 / 2 processes and 1 GPU
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
export OMP_NUM_THREADS=1
show() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step']*1e3,1), {k: (round(v['ms'],2), v['launches']) for k,v in d['profile_ms'].items()})"; }
for N in 4 2; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2991$N bench_config.py --workload rsim --gpus $N > gpurun_out/r${N}_p.json 2> gpurun_out/r${N}_p.err; echo "rsim ${N}p prof rc=$?"; show gpurun_out/r${N}_p.json
done
timeout 300 python bench_config.py --workload rsim --gpus 1 > gpurun_out/r1_p.json 2> gpurun_out/r1_p.err; echo "rsim 1 GPU prof rc=$?"; show gpurun_out/r1_p.json
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29950 tools/trace_rsim.py > gpurun_out/trace_rsim.log 2>&1; echo "trace rc=$?"; tail -30 gpurun_out/trace_rsim.log
