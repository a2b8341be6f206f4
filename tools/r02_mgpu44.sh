# round 2, 2-GPU call 44: the reference arm under torchrun (rank 0 runs it, the others exit 0)
export OMP_NUM_THREADS=1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29944 bench.py --impl reference --gpus 2 --steps 5 --warmup 3 > gpurun_out/ref2.json 2> gpurun_out/ref2.err
echo "reference N=2 rc=$?"; tail -1 gpurun_out/ref2.json | cut -c1-400
