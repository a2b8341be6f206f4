# round 2, GPU call 7: TMA probe again, then the TMA / VMM GPU tests, then the whole -m gpu suite
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
nvcc -gencode arch=compute_100a,code=sm_100a -I include -o tools/tma_copy_probe tools/tma_copy_probe.cu -L paper_2503_10516_b200 -lcel -Xlinker -rpath=$PWD/paper_2503_10516_b200 || exit 1
while read -r shape; do
  [ -z "$shape" ] && continue
  echo "== $shape"; timeout 60 ./tools/tma_copy_probe $shape 2>&1 | tail -2
done <<'SHAPES'
4 66 260 1 66 260 1 1 258 0 1 258 0 65 1 1
4 12 12 1 12 12 1 2 4 0 2 4 0 5 7 1
4 12 12 1 12 16 1 2 4 0 2 4 0 5 8 1
4 12 12 1 12 16 1 2 3 0 2 4 0 5 8 1
4 7 7 8 7 7 8 0 0 4 0 0 4 7 7 4
SHAPES
export CUDA_LAUNCH_BLOCKING=1 CEL_EXEC_THREAD=0
for c in "ws2d_axes 4" "ws2d_box 4 none" "rand1 4 none" "rand5 3 none"; do
  CEL_COPY=tma CEL_NO_GROW=1 timeout 120 python tests/tools/tma_debug.py $c 2>&1 | tail -1
done
unset CUDA_LAUNCH_BLOCKING CEL_EXEC_THREAD
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 -x > gpurun_out/pytest.log 2>&1
echo "pytest all rc=$?"; tail -15 gpurun_out/pytest.log
