"""Peer data movement through the C-ABI on G GPUs of one process (for ncu
NVLink counters and timing):
  python tools/peer_case.py push|mc [G] [MiB]
push: an `all` read of a float4 buffer as G(G-1) peer pushes by the SM copy
kernel (CEL_PEER_DMA=0, collective off); mc: the same set as NVLS multicast
stores (CEL_COLL_MC=1).  Three rounds; prints per-round device time."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
mode = sys.argv[1] if len(sys.argv) > 1 else "push"
G = int(sys.argv[2]) if len(sys.argv) > 2 else 2
mib = int(sys.argv[3]) if len(sys.argv) > 3 else 256
if mode == "push":
    os.environ["CEL_PEER_DMA"] = "0"
else:
    os.environ["CEL_COLL_MC"] = "1"
from paper_2503_10516_b200 import cel  # noqa: E402

N = mib * (1 << 20) // 16
rt = cel.Runtime(G, cuda_devices=list(range(G)), arena_bytes=max(1 << 30, 3 * N * 16), collective=(mode == "mc"))
rt.buffer_create(1, [N], 16)
rt.buffer_create(1, [N], 16)
full = ([0], [N])
produce = cel.task_desc({"dims": 1, "range": full, "kernel": "fill_const", "params": {"value": 1.0},
                         "accesses": [(0, "write", ("one_to_one",))]})
consume = cel.task_desc({"dims": 1, "range": full, "kernel": "fill_const", "params": {"value": 2.0},
                         "accesses": [(1, "write", ("one_to_one",)), (0, "read", ("all",))]})
rt.profile_enable(True)
out = []
for r in range(3):
    rt.submit_desc(produce[0])
    rt.wait()
    t0 = time.perf_counter()
    rt.submit_desc(consume[0])
    rt.wait()
    out.append((time.perf_counter() - t0) * 1e3)
prof = rt.profile_read()
st = rt.stats()
rt.shutdown()
print(json.dumps({"mode": mode, "G": G, "MiB": mib, "host_ms_per_round": out,
                  "profile": {k: {"ms": v[0], "n": v[1]} for k, v in prof.items()},
                  "coll_multicast": st["coll_multicast"], "copies": st["copies_coherence"]}))
