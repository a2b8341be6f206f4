# round 2, 2-GPU call 20: debug the fused RSim row with lookahead none
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
export OMP_NUM_THREADS=1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 120 $TR --master-port 29601 tests/mp_check.py --execute 1 --quick --only rsim --modes none > gpurun_out/mp_rsim_none.log 2>&1
echo "fused none rc=$?"; grep -E "ok|FAIL|MP_CHECK|CelError" gpurun_out/mp_rsim_none.log | head -5
CEL_FUSE_HALO=0 timeout 120 $TR --master-port 29602 tests/mp_check.py --execute 1 --quick --only rsim --modes none > gpurun_out/mp_rsim_none0.log 2>&1
echo "unfused none rc=$?"; grep -E "ok|FAIL|MP_CHECK|CelError" gpurun_out/mp_rsim_none0.log | head -5
CEL_NO_GROW=1 timeout 120 $TR --master-port 29603 tests/mp_check.py --execute 1 --quick --only rsim --modes none > gpurun_out/mp_rsim_none_ng.log 2>&1
echo "fused none nogrow rc=$?"; grep -E "ok|FAIL|MP_CHECK|CelError" gpurun_out/mp_rsim_none_ng.log | head -5
CEL_TRACE=1 timeout 120 $TR --master-port 29604 tests/mp_check.py --execute 1 --quick --only rsim --modes none > gpurun_out/mp_rsim_none_tr.log 2>&1
echo "traced rc=$?"; grep -c "" gpurun_out/mp_rsim_none_tr.log
