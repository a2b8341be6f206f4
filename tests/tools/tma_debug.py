"""Run one program on virtual devices of GPU 0 and compare with the oracle
(debug helper: one program per process, so a sticky CUDA error names it).

  python tests/tools/tma_debug.py <case> [G]      env: CEL_COPY=tma etc. as needed
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.scheduler import Runtime as OracleRuntime  # noqa: E402
from oracle.simulate import simulate  # noqa: E402
from paper_2503_10516_b200 import cel  # noqa: E402
from workloads import programs as P  # noqa: E402
from workloads.driver import run_program  # noqa: E402

CASES = {
    "jac36": lambda: P.jacobi3d(36, 4), "jac20": lambda: P.jacobi3d(20, 3),
    "ws2d_axes": lambda: P.wavesim(515, 5, rows=130, split="2d", mapper="neighborhood_axes"),
    "ws2d_box": lambda: P.wavesim(516, 4, rows=260, split="2d"),
}
for s in range(8):
    CASES["rand%d" % s] = (lambda s=s: P.random_program(7300 + s))

name = sys.argv[1]
G = int(sys.argv[2]) if len(sys.argv) > 2 else 4
mode = sys.argv[3] if len(sys.argv) > 3 else "auto"
prog = CASES[name]()
rt = cel.Runtime(G, cuda_devices=[0] * G, arena_bytes=64 << 20, lookahead=mode)
st = {}
close = rt.shutdown


def shut():
    if rt.h is not None:
        st.update(rt.stats())
    close()


rt.shutdown = shut
got = [r[1] for r in run_program(rt, prog) if r[0] == "read"]
o = OracleRuntime(G, lookahead=mode)
run_program(o, prog)
exp = simulate(o)
bad = 0
for k, arr in enumerate(got):
    d = exp[k] != np.uint32(0x7FC00BAD)
    bad += int((arr[d] != exp[k][d]).sum())
print(json.dumps({"case": name, "G": G, "mode": mode, "mismatches": bad, "tma": st.get("tma_copy_launches"),
                  "copies": st.get("copies_coherence")}))
