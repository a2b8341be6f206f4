# round 2, 2-GPU call 22: fused RSim with growth -- isolate (in-kernel waits off / PDL off), trace
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
export OMP_NUM_THREADS=1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
CEL_HALO_MODE=1 timeout 120 $TR --master-port 29601 tests/mp_check.py --execute 1 --quick --only rsim --modes none > gpurun_out/mp_a.log 2>&1
echo "in-waits off rc=$?"; grep -E " ok|FAIL|MP_CHECK|CelError" gpurun_out/mp_a.log | head -3
CEL_PDL=0 timeout 120 $TR --master-port 29602 tests/mp_check.py --execute 1 --quick --only rsim --modes none > gpurun_out/mp_b.log 2>&1
echo "pdl off rc=$?"; grep -E " ok|FAIL|MP_CHECK|CelError" gpurun_out/mp_b.log | head -3
CEL_TRACE=1 timeout 120 $TR --master-port 29604 tests/mp_check.py --execute 1 --quick --only rsim --modes none > gpurun_out/mp_tr.log 2>&1
echo "traced rc=$?"; grep -E "rsim fused|push iid" gpurun_out/mp_tr.log | head -12
