"""Diagnostic: library per-launch profile vs wall-clock per step (Jacobi and WaveSim)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2503_10516_b200 import cel
from workloads import programs as P

def run(kind, steps, profile):
    if kind == "jacobi":
        n = 1024
        rt = cel.Runtime(1, arena_bytes=int(2 * n ** 3 * 4 * 1.05) + (512 << 20))
        rt.buffer_create(3, [n] * 3, 4); rt.buffer_create(3, [n] * 3, 4)
        rt.task_submit(P.jacobi3d(n, 1)["ops"][0][1])
        d = [cel.task_desc(P.jacobi_step(n, k)[1]) for k in (0, 1)]
        name = "jacobi7"
    else:
        n = 16384
        rt = cel.Runtime(1, arena_bytes=int(2 * (n + 2) * n * 4 * 1.05) + (512 << 20))
        rt.buffer_create(2, [n, n], 4); rt.buffer_create(2, [n, n], 4)
        for op in P.wavesim_init(n): rt.task_submit(op[1])
        d = [cel.task_desc(P.wavesim_step(n, k)[1]) for k in (0, 1)]
        name = "wave5"
    for k in range(6): rt.submit_desc(d[k % 2][0])
    rt.wait()
    rt.profile_enable(profile)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); t0 = time.perf_counter()
    for k in range(steps): rt.submit_desc(d[k % 2][0])
    t1 = time.perf_counter()
    rt.wait(); e1.record(); torch.cuda.synchronize()
    prof = rt.profile_read() if profile else {}
    rt.shutdown()
    ms = e0.elapsed_time(e1)
    print("%-7s profile=%d steps=%d wall %.3f ms/step  submit %.1f us/step  profile %s" % (
        kind, profile, steps, ms / steps, (t1 - t0) / steps * 1e6,
        {k: round(v[0] / v[1], 4) for k, v in prof.items()}))

for kind in ("jacobi", "wave"):
    for profile in (False, True):
        run(kind, 50 if kind == "jacobi" else 200, profile)
