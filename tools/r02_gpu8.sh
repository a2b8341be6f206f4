# round 2, GPU call 8: TMA alignment rule, then the whole -m gpu suite, bench copy block
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
nvcc -gencode arch=compute_100a,code=sm_100a -I include -o tools/tma_copy_probe tools/tma_copy_probe.cu -L paper_2503_10516_b200 -lcel -Xlinker -rpath=$PWD/paper_2503_10516_b200 || exit 1
for shape in "4 12 12 1 12 16 1 2 3 0 2 4 0 5 8 1" "4 12 12 1 12 16 1 2 4 0 2 4 0 5 8 1" "4 20 20 36 20 20 36 1 1 0 1 19 0 18 1 36"; do
  echo "== $shape"; timeout 60 ./tools/tma_copy_probe $shape 2>&1 | tail -2
done
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest.log 2>&1
echo "pytest all rc=$?"; tail -15 gpurun_out/pytest.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_k20.json 2> gpurun_out/bench_k20.err
echo "bench rc=$?"; cat gpurun_out/bench_k20.json
