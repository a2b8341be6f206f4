"""Virtual-node mode measurement: the paper's multi-node
lowering -- push / await-push -> staging copy into pinned host memory (M1),
send, receive (pilots + receive arbitration), copy to the device -- on one box,
N nodes x D devices in one process, against the single-node runtime over the
same N*D GPUs (peer pushes over NVLink, no staging).  Timed between two epochs
(host clock around cel_wait: every node's GPU work is inside), so it includes
the host-side arbitration.

  python bench_nodes.py --nodes 2 --devices-per-node 1 [--workload wavesim|nbody] [--steps K]
"""

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2503_10516_b200 import cel  # noqa: E402
from workloads import programs as P  # noqa: E402


def run(nodes, D, workload, steps, warmup, n):
    G = nodes * D
    devs = list(range(G))
    rt = cel.Runtime(D, cuda_devices=devs, arena_bytes=(4 << 30), n_nodes=nodes) if nodes > 1 else \
        cel.Runtime(G, cuda_devices=devs, arena_bytes=(4 << 30))
    if workload == "wavesim":
        rt.buffer_create(2, [n, n], 4)
        rt.buffer_create(2, [n, n], 4)
        for op in P.wavesim_init(n, 2):
            rt.task_submit(op[1])
        descs = [cel.task_desc(P.wavesim_step(n, k)[1]) for k in (0, 1)]

        def step(s):
            rt.submit_desc(descs[s % 2][0])
    else:
        prog = P.nbody(n, 1)
        rt.buffer_create(1, [n], 16)
        rt.buffer_create(1, [n], 16)
        for op in prog["ops"][:2]:
            rt.task_submit(op[1])
        descs = [cel.task_desc(op[1]) for op in prog["ops"][2:4]]

        def step(s):
            rt.submit_desc(descs[0][0])
            rt.submit_desc(descs[1][0])
    for s in range(warmup):
        step(s)
    rt.wait()
    st0 = rt.stats()
    t0 = time.perf_counter()
    for s in range(steps):
        step(warmup + s)
    rt.wait()
    dt = time.perf_counter() - t0
    st1 = rt.stats()
    rt.shutdown()
    d = {k: st1[k] - st0[k] for k in ("n_send", "n_receive", "n_split_receive", "n_await_receive", "pulls",
                                       "pull_bytes", "copies_coherence", "bytes_coherence", "bytes_d2d_peer",
                                       "staging_elided", "staging_materialized")}
    return {"nodes": nodes, "devices_per_node": D, "gpus": G, "workload": workload, "n": n, "steps": steps,
            "steps_per_s": steps / dt, "ms_per_step": dt * 1e3 / steps,
            "sends_per_step": d["n_send"] / steps, "pull_bytes_per_step": d["pull_bytes"] / steps,
            "pull_GBps": d["pull_bytes"] / dt / 1e9, "peer_bytes_per_step": d["bytes_d2d_peer"] / steps,
            "staging_copies_elided_per_step": d["staging_elided"] / steps,
            "staging_copies_executed_late_per_step": d["staging_materialized"] / steps,
            "direct_sends": os.environ.get("CEL_DIRECT_SENDS", "1") != "0"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nodes", type=int, default=2)
    ap.add_argument("--devices-per-node", type=int, default=1)
    ap.add_argument("--workload", default="wavesim", choices=["wavesim", "nbody"])
    ap.add_argument("--steps", type=int, default=0)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--n", type=int, default=0)
    a = ap.parse_args()
    n = a.n or (16384 if a.workload == "wavesim" else 1 << 20)
    steps = a.steps or (200 if a.workload == "wavesim" else 3)
    out = {"virtual_nodes": run(a.nodes, a.devices_per_node, a.workload, steps, a.warmup, n),
           "single_node": run(1, a.nodes * a.devices_per_node, a.workload, steps, a.warmup, n)}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
