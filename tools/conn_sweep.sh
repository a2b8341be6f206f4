# WaveSim bench at N GPUs with CUDA_DEVICE_MAX_CONNECTIONS = 8 (default) and 32
N=${1:-4}
for c in 8 32; do
  CUDA_DEVICE_MAX_CONNECTIONS=$c timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
    --master-addr 127.0.0.1 --master-port 28${N}$c bench.py --gpus $N --steps 3000 --warmup 20 \
    --no-cpu-baseline --no-e2e 2>/dev/null | grep "^{" > gpurun_out/conn_${N}_$c.json
  python - "$c" "$N" <<'PY'
import json, sys
c, n = sys.argv[1], sys.argv[2]
d = json.load(open("gpurun_out/conn_%s_%s.json" % (n, c)))
print("N=%s connections=%s value=%.1f ms/step=%.4f kernel_share=%.3f" % (n, c, d["value"], d["ms_per_step"], d["roofline"]["kernel_share_of_step"]))
PY
done
