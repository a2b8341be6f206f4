# round 2, 2-GPU call 21: compute-sanitizer on the fused RSim row with growth (lookahead none)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
export OMP_NUM_THREADS=1
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 --no-python \
  /usr/local/cuda/bin/compute-sanitizer --tool memcheck --print-limit 5 python tests/mp_check.py --execute 1 --quick --only rsim --modes none > gpurun_out/san_rsim.log 2>&1
echo "sanitizer rc=$?"; grep -E "Invalid|Error|error|at 0x|by thread|Address|kernel|=========" gpurun_out/san_rsim.log | head -40
