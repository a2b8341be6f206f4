"""Small programs for compute-sanitizer runs (memcheck / racecheck / synccheck):
every kernel family, resize copies, d2d copies between virtual devices, the
shell/interior split, TMA Jacobi, H2D/D2H."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from paper_2503_10516_b200 import cel
from oracle.scheduler import Runtime as ORt
from workloads.driver import run_program
from oracle.simulate import simulate
from workloads import programs as P
progs = [P.c1_chain(1024), P.wavesim(1024, 4, rows=700), P.jacobi3d(72, 2), P.nbody(600, 1, host_init=True),
         P.rsim(1000, 12), P.random_program(3), P.random_program(4)]
bad = 0
for prog in progs:
    for mode in ("auto", "none"):
        rt = cel.Runtime(3, cuda_devices=[0, 0, 0], lookahead=mode, arena_bytes=64 << 20)
        got = [r[1] for r in run_program(rt, prog) if r[0] == "read"]
        o = ORt(3, lookahead=mode); run_program(o, prog); exp = simulate(o)
        for k, g in enumerate(got):
            d = exp[k] != np.uint32(0x7FC00BAD)
            if not np.array_equal(g[d], exp[k][d]): bad += 1
print("SANITIZE_PROGRAMS", "PASS" if bad == 0 else "FAIL %d" % bad)
