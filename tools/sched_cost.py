"""Host cost of IDAG generation per WaveSim step (execute=0: no GPU touched), G = 1, 2, 4, 8,
through the Python binding.  CEL_SCHED_MEMO=0 switches the steady-state compile memo off;
tools/sched_prof.cpp measures the scheduler alone (no Python)."""
import sys, time
sys.path.insert(0, "/root/repo")
from paper_2503_10516_b200 import cel
from workloads import programs as P
for G in (1, 2, 4, 8):
    rt = cel.Runtime(G, execute=False)
    n = 16384
    rt.buffer_create(2, [n, n], 4); rt.buffer_create(2, [n, n], 4)
    prog = P.wavesim(n, 4)
    for op in prog["ops"][:2]:
        rt.task_submit(op[1])
    descs = [cel.task_desc(P.wavesim_step(n, k)[1]) for k in (0, 1)]
    for s in range(100): rt.submit_desc(descs[s % 2][0])
    rt.wait()
    t0 = time.perf_counter(); K = 3000
    for s in range(K): rt.submit_desc(descs[s % 2][0])
    rt.wait()
    dt = time.perf_counter() - t0
    st = rt.stats()
    print(G, "%.1f us/step" % (dt / K * 1e6), "memo hits %d misses %d" % (st["memo_hits"], st["memo_misses"]))
    rt.shutdown()
