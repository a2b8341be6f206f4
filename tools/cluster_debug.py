"""Virtual-node debug run: one program on N nodes x D devices, instruction trace on stderr."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_10516_b200 import cel
from workloads.driver import run_program
from workloads import programs as P
name, N, D, mode = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
prog = {"c1": lambda: P.c1_chain(256), "ws": lambda: P.wavesim(256, 7, rows=96), "nbody": lambda: P.nbody(300, 2),
        "fig4": lambda: P.nbody(256, 2, host_init=True), "jac": lambda: P.jacobi3d(20, 3),
        "rsim": lambda: P.rsim(256, 12)}[name]()
rt = cel.Runtime(D, cuda_devices=[0] * (N * D), lookahead=mode, arena_bytes=64 << 20, n_nodes=N,
                 instr_log_path="gpurun_out/dbg.jsonl")
print("created", flush=True)
res = run_program(rt, prog)
print("done", len(res), flush=True)
