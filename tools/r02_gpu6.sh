# round 2, GPU call 6: TMA copy kernel probe on single box shapes (one process each)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
nvcc -gencode arch=compute_100a,code=sm_100a -I include -o tools/tma_copy_probe tools/tma_copy_probe.cu -L paper_2503_10516_b200 -lcel -Xlinker -rpath=$PWD/paper_2503_10516_b200 || exit 1
while read -r shape; do
  [ -z "$shape" ] && continue
  echo "== $shape"; timeout 60 ./tools/tma_copy_probe $shape 2>&1 | tail -3
done <<'SHAPES'
4 20 20 36 20 20 36 1 1 0 1 19 0 18 1 36
4 66 260 1 66 260 1 1 258 0 1 258 0 65 1 1
4 66 260 1 66 264 1 1 3 0 1 3 0 65 1 1
4 66 260 1 66 264 1 1 7 0 1 7 0 65 2 1
4 66 260 1 66 264 1 0 0 0 0 4 0 66 100 1
4 7 7 8 7 7 8 1 2 3 2 1 0 3 2 5
4 7 7 8 7 7 8 0 0 4 0 0 4 7 7 4
4 12 12 1 12 12 1 2 4 0 2 4 0 5 7 1
4 12 12 1 12 16 1 2 4 0 2 4 0 5 7 1
4 40 1 1 40 1 1 3 0 0 3 0 0 10 1 1
SHAPES
