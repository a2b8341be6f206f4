"""Find virtual-node programs that hang or mismatch with device-direct sends:
one subprocess per (seed, N, D, mode), 60 s each.  Prints one line per case."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
CHILD = r'''
import os, sys, json
sys.path.insert(0, %r)
import numpy as np
from oracle.cluster import Cluster
from oracle.simulate import GARBAGE, simulate_cluster
from paper_2503_10516_b200 import cel
from workloads import programs as P
from workloads.driver import run_program
seed, N, D, mode, step = %d, %d, %d, %r, %d
prog = P.random_program(seed)
rt = cel.Runtime(D, cuda_devices=[0] * (N * D), lookahead=mode, arena_bytes=64 << 20, n_nodes=N, horizon_step=step)
got = [r[1] for r in run_program(rt, prog) if r[0] == "read"]
o = Cluster(N, D, lookahead=mode, horizon_step=step)
run_program(o, prog)
exp = simulate_cluster(o)
bad = sum(int(((a != exp[k]) & (exp[k] != GARBAGE)).sum()) for k, a in enumerate(got))
print("RESULT", bad)
'''
out = []
for s in range(int(sys.argv[2]) if len(sys.argv) > 2 else 0, int(sys.argv[1]) if len(sys.argv) > 1 else 30):
    for N, D in ((2, 1), (2, 2), (3, 1), (3, 2)):
        mode = ["none", "auto", "infinite"][s % 3]
        seed = 6100 + 11 * N + D + s
        env = dict(os.environ, CEL_DIRECT_SENDS=os.environ.get("PROBE_DIRECT", "1"))
        try:
            step = 2 + s % 3 if os.environ.get("PROBE_STEP") == "test" else int(os.environ.get("PROBE_STEP", "4"))
            r = subprocess.run([sys.executable, "-c", CHILD % (ROOT, seed, N, D, mode, step)], capture_output=True, text=True,
                               timeout=60, env=env)
            res = [l for l in r.stdout.splitlines() if l.startswith("RESULT")]
            status = ("mismatch %s" % res[0].split()[1]) if res and res[0].split()[1] != "0" else ("ok" if res else "error " + r.stderr[-200:].replace("\n", " "))
        except subprocess.TimeoutExpired:
            status = "HANG"
        if status != "ok" or os.environ.get("PROBE_ALL"):
            print(json.dumps({"seed": seed, "N": N, "D": D, "mode": mode, "status": status}), flush=True)
print("done", flush=True)
