"""wave5 kernel time per launch on one GPU for a rows x 16384 chunk (the per-
device chunk of WaveSim 16384^2 at G = 16384 / rows), CUDA-event profile.
  CEL_WAVE_STRIP=h python tools/wave_strip.py rows"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2503_10516_b200 import cel  # noqa: E402
from workloads import programs as P  # noqa: E402

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
n = 16384
rt = cel.Runtime(1, arena_bytes=2 * rows * n * 4 + (256 << 20))
rt.buffer_create(2, [rows, n], 4)
rt.buffer_create(2, [rows, n], 4)
for op in P.wavesim_init(n, rows=rows):
    rt.task_submit(op[1])
d = [cel.task_desc(P.wavesim_step(n, k, rows=rows)[1]) for k in (0, 1)]
for k in range(20):
    rt.submit_desc(d[k % 2][0])
rt.wait()
rt.profile_enable(True)
K = 400
for k in range(K):
    rt.submit_desc(d[k % 2][0])
rt.wait()
ms, cnt = rt.profile_read()["wave5"]
rt.shutdown()
us = ms / cnt * 1e3
print(json.dumps({"rows": rows, "strip": os.environ.get("CEL_WAVE_STRIP", "auto"), "us_per_launch": us,
                  "GBps": 12 * rows * n / (us / 1e6) / 1e9}))
