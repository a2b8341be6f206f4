# build + smoke + GPU tests + bench N=1 / 2 / 4 (round-end rehearsal)
mkdir -p gpurun_out/final2
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -1
timeout 400 python bench.py > gpurun_out/final2/bench_n1.json 2> gpurun_out/final2/bench_n1.err
for N in 2 4; do
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port 2955$N bench.py --gpus $N --steps 4000 --warmup 20 2>/dev/null | grep "^{" > gpurun_out/final2/bench_n$N.json
done
timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29562 \
  bench.py --impl reference --gpus 2 --steps 3 --warmup 3 2>/dev/null | grep "^{" | cut -c1-160
for N in 1 2 4; do
  python -c "import json; d=json.loads(open('gpurun_out/final2/bench_n$N.json').read().strip().splitlines()[-1]); print('N=$N', round(d['value'], 1), 'frac', round(d['roofline']['frac'], 3), 'e2e', d['e2e'] and round(d['e2e']['value'], 1), 'clocks', d['clocks'])"
done
