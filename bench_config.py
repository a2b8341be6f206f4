"""Multi-GPU measurement of the other BASELINE configs with bench.py's protocol
(one process per GPU under torchrun, barrier + synchronize around the timed
region, CUDA events, max over ranks).  Prints one JSON line on rank 0.

  python bench_config.py --workload jacobi3d|nbody|rsim --gpus N [--steps K] [--warmup W]
                         [--fast-math] [--lookahead auto|none]

  jacobi3d  C5: 1024^3 fp32 7-point, 2-D split (z, y), strided y-face halos
  nbody     C3: 2^20 float4 bodies, 'all' read of P -> G(G-1) peer pushes per step
  rsim      C4: W = 84,000, T rows (default 1024): whole program timed (value = rows/s)
  gather    C3's communication stage alone: every step rewrites P (2^20 float4 = 16 MiB) on
            its owners and runs a task reading it through `all`, i.e. one all-gather set of
            G (G-1) copies; value = gathers/s, GB/s received per device vs NVLink
"""

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2503_10516_b200 import cel  # noqa: E402
from workloads import programs as P  # noqa: E402

FP32_NOMINAL_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", required=True, choices=["jacobi3d", "nbody", "rsim", "wavesim", "gather"])
    ap.add_argument("--split", default="1d", help="wavesim: 1d | 2d")
    ap.add_argument("--mapper", default="neighborhood", help="wavesim: neighborhood | neighborhood_axes")
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=0)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--fast-math", action="store_true")
    ap.add_argument("--lookahead", default="auto")
    ap.add_argument("--rows", type=int, default=1024)
    ap.add_argument("--collective", type=int, default=1, help="1: all-gather copy sets as NCCL broadcasts")
    args = ap.parse_args()
    rank, world, local = bench.env_rank()
    G = args.gpus
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")
    torch.cuda.set_device(local if world > 1 else 0)
    peak, peak_kind = bench.measured_peaks()

    if args.workload == "jacobi3d":
        n = 1024
        steps = args.steps or 200
        arena = int(2 * n ** 3 * 4 / G * 1.2) + (1 << 30)
        rt = bench.make_runtime(cel, G, rank, world, dist, arena)
        rt.buffer_create(3, [n, n, n], 4)
        rt.buffer_create(3, [n, n, n], 4)
        rt.task_submit(P.jacobi3d(n, 1)["ops"][0][1])
        descs = [cel.task_desc(P.jacobi_step(n, k)[1]) for k in (0, 1)]
        submit = lambda s: rt.submit_desc(descs[s % 2][0])  # noqa: E731
        kernel = "jacobi7"
    elif args.workload == "wavesim":
        # NEXT-3 variants of C2: 2-D split and the axis-only neighbourhood
        n = 16384
        steps = args.steps or 1000
        arena = int(2 * n * n * 4 / G * 1.1) + (1 << 30)
        rt = bench.make_runtime(cel, G, rank, world, dist, arena)
        rt.buffer_create(2, [n, n], 4)
        rt.buffer_create(2, [n, n], 4)
        for op in P.wavesim_init(n, split=args.split):
            rt.task_submit(op[1])
        descs = [cel.task_desc(P.wavesim_step(n, k, split=args.split, mapper=args.mapper)[1]) for k in (0, 1)]
        submit = lambda s: rt.submit_desc(descs[s % 2][0])  # noqa: E731
        kernel = "wave5"
    elif args.workload == "nbody":
        N = 1 << 20
        steps = args.steps or 3
        rt = bench.make_runtime(cel, G, rank, world, dist, 1 << 30, fast_math=args.fast_math,
                                collective=bool(args.collective))
        prog = P.nbody(N, 1)
        rt.buffer_create(1, [N], 16)
        rt.buffer_create(1, [N], 16)
        for op in prog["ops"][:2]:
            rt.task_submit(op[1])
        descs = [cel.task_desc(op[1]) for op in prog["ops"][2:4]]

        def submit(s):
            rt.submit_desc(descs[0][0])
            rt.submit_desc(descs[1][0])
        kernel = "nbody_step"
    elif args.workload == "gather":
        N = 1 << 20
        steps = args.steps or 200
        rt = bench.make_runtime(cel, G, rank, world, dist, 1 << 30, collective=bool(args.collective))
        rt.buffer_create(1, [N], 16)
        rt.buffer_create(1, [N], 16)
        full = ([0], [N])
        # the owners rewrite P, then a task declares an `all` read of P (its kernel
        # writes V only): the coherence diff makes that read one all-gather set
        produce = cel.task_desc({"dims": 1, "range": full, "kernel": "fill_const", "params": {"value": 1.0},
                                 "accesses": [(0, "write", ("one_to_one",))]})
        consume = cel.task_desc({"dims": 1, "range": full, "kernel": "fill_const", "params": {"value": 2.0},
                                 "accesses": [(1, "write", ("one_to_one",)), (0, "read", ("all",))]})

        def submit(s):
            rt.submit_desc(produce[0])
            rt.submit_desc(consume[0])
        kernel = "fill_const"
    else:
        W, T = 84000, args.rows
        steps = T
        rt = bench.make_runtime(cel, G, rank, world, dist, 4 << 30, lookahead=args.lookahead,
                                collective=bool(args.collective))
        prog = P.rsim(W, T)
        rt.buffer_create(2, [T, W], 4)
        descs = [cel.task_desc(op[1]) for op in prog["ops"] if op[0] == "task"]
        submit = lambda s: rt.submit_desc(descs[s][0])  # noqa: E731
        kernel = "rsim_row"

    if args.workload != "rsim":
        for s in range(args.warmup):
            submit(s)
    rt.wait()
    st0 = rt.stats()
    prof_on = not os.environ.get("CEL_BENCH_NOPROF")     # per-launch events cost host time (RSim: host-bound)
    if prof_on:
        rt.profile_enable(True)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    t0 = time.perf_counter()
    for s in range(steps):
        submit(s if args.workload == "rsim" else args.warmup + s)
    rt.wait()
    e1.record()
    torch.cuda.synchronize()
    host_s = time.perf_counter() - t0
    if dist:
        dist.barrier()
    ms = e0.elapsed_time(e1)
    prof = rt.profile_read()
    st1 = rt.stats()
    if dist:
        t = torch.tensor([ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    rt.wait()
    if dist:
        dist.barrier()
    rt.shutdown()
    km = prof.get(kernel, (0.0, 0))[0] + prof.get("shell", (0.0, 0))[0]
    line = {"workload": args.workload, "n_gpus": G, "processes": world, "steps": steps,
            "value": steps / (ms / 1e3), "unit": "rows/s" if args.workload == "rsim" else "steps/s",
            "ms_per_step": ms / steps, "host_ms_per_step": host_s * 1e3 / steps,
            "gen_us_per_step": (st1["gen_ns"] - st0["gen_ns"]) / 1e3 / steps,
            "exec_us_per_step": {k[8:]: (st1[k] - st0[k]) / 1e3 / steps for k in
                                 ("exec_ns_alloc", "exec_ns_free", "exec_ns_copy", "exec_ns_kernel", "exec_ns_horizon",
                                  "exec_ns_epoch")},
            "host_us_per_step": {k: (st1[k] - st0[k]) / 1e3 / steps for k in ("signal_ns", "remote_wait_ns")},
            "per_step": {k: (st1[k] - st0[k]) / steps for k in ("signals", "remote_waits", "event_waits",
                                                                   "kernel_launches", "copy_launches", "memcpy_calls")},
            "coll_p2p": st1["coll_p2p"] - st0["coll_p2p"],
            "gpu_launches": st1["kernel_launches"] - st0["kernel_launches"],
            "collective": bool(args.collective),
            "coll_groups": st1["coll_groups"] - st0["coll_groups"],
            "coll_allgathers": st1["coll_allgathers"] - st0["coll_allgathers"],
            "profile_ms": {k: {"ms": v[0], "launches": v[1]} for k, v in prof.items()}}
    if args.workload == "jacobi3d" and km > 0:   # (per-launch profiling off, CEL_BENCH_NOPROF: no roofline)
        cells = 1024 ** 3 / G
        line["roofline"] = {"bound": "hbm", "unit": "GB/s", "peak": peak, "peak_source": peak_kind,
                            "achieved": 8 * cells / (km / 1e3 / steps) / 1e9,
                            "note": "rank-0 chunk; kernel time = interior + shell launch durations (they overlap, so this is a lower bound)"}
        line["roofline"]["frac"] = line["roofline"]["achieved"] / peak
    elif args.workload == "jacobi3d":
        pass
    elif args.workload == "nbody" and km > 0:
        inter = (1 << 20) * (1 << 20) / G * steps
        line["roofline"] = {"bound": "alu", "unit": "TFLOP/s", "peak": FP32_NOMINAL_TFLOPS,
                            "achieved": 20 * inter / (km / 1e3) / 1e12, "fast_math": args.fast_math}
        line["roofline"]["frac"] = line["roofline"]["achieved"] / FP32_NOMINAL_TFLOPS
        line["interactions_per_s"] = (1 << 40) * steps / (ms / 1e3)
    elif args.workload == "nbody":
        line["interactions_per_s"] = (1 << 40) * steps / (ms / 1e3)
    elif args.workload == "wavesim":
        line["split"] = args.split
        line["mapper"] = args.mapper
        line["coherence_copies_per_step"] = (st1["copies_coherence"] - st0["copies_coherence"]) / steps
    elif args.workload == "gather":
        recv = (G - 1) / G * 16 * (1 << 20)
        line["gather_bytes_received_per_device"] = recv
        line["GBps_received_per_device"] = recv / (ms / 1e3 / steps) / 1e9
        line["frac_nvlink_measured_ref"] = line["GBps_received_per_device"] / 770.0
        line["coll_multicast"] = st1["coll_multicast"] - st0["coll_multicast"]
        line["gather_sets"] = st1["gather_sets"] - st0["gather_sets"]
        line["note"] = "step = rewrite P (fill kernel) + the gather; the fill's ~5 us is inside ms_per_step"
    else:
        line["lookahead"] = args.lookahead
        line["alloc"] = st1["n_alloc"] - st0["n_alloc"]
        line["resize_copies"] = st1["copies_resize"] - st0["copies_resize"]
        line["resize_copies_elided"] = st1["copies_elided"] - st0["copies_elided"]
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
