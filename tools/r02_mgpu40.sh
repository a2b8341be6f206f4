# round 2, 4-GPU call 40: regression sweep against the earlier round-2 profiles -- suite (1 GPU), configs at 4 GPUs
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
export OMP_NUM_THREADS=1
timeout 900 python bench_suite.py > gpurun_out/suite.json 2> gpurun_out/suite.err
echo "suite rc=$?"; python - <<'PY'
import json
d=json.load(open("gpurun_out/suite.json"))
print("c1", {k: round(v["us_per_task"],1) for k,v in d["c1"].items() if isinstance(v, dict)})
print("c3", round(d["c3"]["steps_per_s"],3), "c3fast", round(d["c3fast"]["steps_per_s"],3))
print("c4", {k: (round(v.get("rows_per_s",0)) if isinstance(v,dict) else v) for k,v in d["c4"].items()})
print("c5", {k: (round(v,1) if isinstance(v,(int,float)) else v) for k,v in d["c5"].items() if not isinstance(v,(dict,list))})
PY
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
for W in jacobi3d nbody; do
  timeout 600 $TR --master-port 29931 bench_config.py --workload $W --gpus 4 > gpurun_out/c4_$W.json 2> gpurun_out/c4_$W.err
  echo "$W 4p rc=$?"; tail -1 gpurun_out/c4_$W.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],2), round(d['ms_per_step'],3))"
done
timeout 600 $TR --master-port 29932 bench_config.py --workload nbody --gpus 4 --fast-math > gpurun_out/c4_nbf.json 2> gpurun_out/c4_nbf.err
echo "nbody fast 4p rc=$?"; tail -1 gpurun_out/c4_nbf.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],2))"
