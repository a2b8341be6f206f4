"""Break the bench's e2e time into its parts (diagnostic, not a bench line)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2503_10516_b200 import cel
from workloads import programs as P
n = 16384
rng = np.random.default_rng(2)
hu = torch.from_numpy(rng.uniform(-1, 1, (n, n)).astype(np.float32)).pin_memory().numpy()
hup = torch.from_numpy(hu.copy()).pin_memory().numpy()
res = torch.empty((n, n), dtype=torch.float32).pin_memory().numpy()
torch.cuda.synchronize()
T = {}
t = time.perf_counter(); rt = cel.Runtime(1, arena_bytes=int(2 * (n + 2) * n * 4 * 1.05) + (512 << 20)); T["create"] = time.perf_counter() - t
t = time.perf_counter(); b0 = rt.buffer_create(2, [n, n], 4, host_init=hu, borrow=True); b1 = rt.buffer_create(2, [n, n], 4, host_init=hup, borrow=True); T["buffers"] = time.perf_counter() - t
d = [cel.task_desc(P.wavesim_step(n, k)[1]) for k in (0, 1)]
t = time.perf_counter(); rt.submit_desc(d[0][0]); rt.wait(); T["first step (allocs + 2 GiB H2D)"] = time.perf_counter() - t
t = time.perf_counter()
for s in range(1, 1001): rt.submit_desc(d[s % 2][0])
rt.wait(); T["1000 steps"] = time.perf_counter() - t
t = time.perf_counter(); rt.buffer_read(b0, ([0, 0], [n, n]), out=res.reshape(n, n, 1, 1).view(np.uint32)); T["readback 1 GiB D2H"] = time.perf_counter() - t
t = time.perf_counter(); rt.shutdown(); T["shutdown"] = time.perf_counter() - t
for k, v in T.items(): print("%-36s %8.1f ms" % (k, v * 1e3))
