# round 2, 4-GPU call 31: final -- suite on 4 GPUs, bench N=1 (driver defaults and K=1000), reference arm, N=2/3/4, launch list
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
export OMP_NUM_THREADS=1
timeout 1500 python -m pytest tests -m gpu -q --timeout 400 --timeout-method thread > gpurun_out/pytest4.log 2>&1
echo "pytest all (4 GPUs) rc=$?"; tail -2 gpurun_out/pytest4.log; grep -E "^E |^FAILED" gpurun_out/pytest4.log | head -20
timeout 900 python bench.py > gpurun_out/final_n1_default.json 2> gpurun_out/final_n1_default.err
echo "bench default rc=$?"; tail -1 gpurun_out/final_n1_default.json | cut -c1-300
timeout 600 python bench.py --steps 1000 --warmup 20 > gpurun_out/final_n1_k1000.json 2> gpurun_out/final_n1_k1000.err
echo "bench K=1000 rc=$?"; tail -1 gpurun_out/final_n1_k1000.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['e2e']['value'], d['clocks'])"
timeout 900 python bench.py --impl reference > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err
echo "reference rc=$?"; tail -1 gpurun_out/final_ref.json | cut -c1-300
for N in 2 3 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2990$N bench.py --gpus $N --steps 1000 --warmup 20 > gpurun_out/final_n$N.json 2> gpurun_out/final_n$N.err
  echo "bench N=$N rc=$?"; tail -1 gpurun_out/final_n$N.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['kernel'], d['roofline']['frac'], d['roofline']['kernel_share_of_step'], d['clocks']['reasons'], d['e2e']['value'] if d.get('e2e') else None)"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final_launches_n1.csv python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-copy > gpurun_out/final_ncu.log 2>&1
echo "ncu launch list rc=$?"; grep -c wave5 gpurun_out/final_launches_n1.csv
