"""Measurement suite for the other SURVEY §8 rows (the contract bench is bench.py).

  python bench_suite.py [--only c1,c3,c4,c5,copy] [--out profiles/rNN_suite.json]

Every number is device time from CUDA events (whole region between two
epochs) or the library's per-launch CUDA-event profile (cel_profile_*), on
the configs of BASELINE.json with synthetic inputs (workloads/programs.py):

  c1    1-D 4096 f32 4-task chain on 2 devices: us per task, instruction counts
  c3    N-body 2^20 float4, 'all' gather as peer coherence copies: steps/s,
        interactions/s, ALU roofline
  c4    RSim-shaped growth W=84,000 x T rows: lookahead auto vs none, resize-copy GB/s
  c5    3-D 7-point 1024^3 f32: steps/s, HBM roofline
  copy  coherence-copy kernel sweep: 1 GiB resize (HBM), strided 2-D resize,
        peer pushes over NVLink (needs 2 GPUs)
"""

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2503_10516_b200 import cel  # noqa: E402
from workloads import programs as P  # noqa: E402

HBM = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
NVLINK_NOMINAL = 900.0      # GB/s per direction
NVLINK_MEASURED_REF = 770.0  # B200_PROFILING.md: measured peer copy per direction
FP32_NOMINAL_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12


def timed(rt, fn):
    rt.wait()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    rt.wait()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 1e3


def c1():
    n_dev = 2
    devs = [0, 1] if torch.cuda.device_count() >= 2 else [0, 0]
    out = {}
    for mode in ("auto", "none"):
        rt = cel.Runtime(n_dev, cuda_devices=devs, lookahead=mode, arena_bytes=64 << 20)
        prog = P.c1_chain(4096)
        a = rt.buffer_create(1, [4096], 4)
        b = rt.buffer_create(1, [4096], 4)
        tasks = [cel.task_desc(op[1]) for op in prog["ops"] if op[0] == "task"]
        reps = 200
        # the 4-task chain, repeated; every task reads a neighbourhood -> 2 halo copies
        dt = timed(rt, lambda: [rt.submit_desc(t[0]) for _ in range(reps) for t in tasks])
        st = rt.stats()
        rt.shutdown()
        out[mode] = {"us_per_task": dt / (reps * 4) * 1e6, "devices": devs,
                     "alloc": st["n_alloc"], "resize_copies": st["copies_resize"],
                     "coherence_copies": st["copies_coherence"], "kernels": st["n_kernel"]}
    return out


def c3(steps=2, fast=False):
    N = 1 << 20
    G = 1
    rt = cel.Runtime(G, arena_bytes=1 << 30, fast_math=fast)
    prog = P.nbody(N, steps=1)
    Pb = rt.buffer_create(1, [N], 16)
    Vb = rt.buffer_create(1, [N], 16)
    for op in prog["ops"][:2]:
        rt.task_submit(op[1])
    step = [cel.task_desc(op[1]) for op in prog["ops"][2:4]]
    rt.submit_desc(step[0][0])
    rt.submit_desc(step[1][0])            # warm-up step
    rt.profile_enable(True)
    dt = timed(rt, lambda: [rt.submit_desc(s[0]) for _ in range(steps) for s in step])
    prof = rt.profile_read()
    rt.shutdown()
    inter = float(N) * N * steps
    flops = 20.0 * inter   # 3 sub, 3 mul + 2 add (r2), add eps, sqrt, div, 2 mul, 3 mul + 3 add
    km = prof.get("nbody_step", (0, 0))[0] / 1e3
    return {"steps_per_s": steps / dt, "interactions_per_s": inter / dt,
            "roofline": {"bound": "alu", "achieved": flops / km / 1e12 if km else None, "unit": "TFLOP/s",
                         "peak": FP32_NOMINAL_TFLOPS, "peak_source": "nominal 148 SM x 128 FP32 lanes x 2 x 1.965 GHz "
                         "(the kernel is built with -fmad=false and IEEE div/sqrt for bit-exact parity: no FMA)",
                         "frac": (flops / km / 1e12 / FP32_NOMINAL_TFLOPS) if km else None,
                         "flop_per_interaction": 20},
            "profile_ms": {k: v[0] for k, v in prof.items()}, "n": N, "devices": G, "fast_math": fast}


def c3fast():
    r = c3(steps=4, fast=True)
    r["roofline"]["peak_source"] = "nominal 148 SM x 128 FP32 lanes x 2 x 1.965 GHz (fast_math: FMA + MUFU rsqrt)"
    return r


def c4(T=1024, W=84000):
    res = {}
    # "none" without in-place growth is the paper's comparison (resize chains
    # executed); "none_grow" shows what the executor's growth recovers
    # none_grow: in-place growth as configured (arena extension, else VMM
    # mapping in one process); none_grow_arena: arena extension only
    for label, mode, grow in (("auto", "auto", True), ("none", "none", False), ("none_grow", "none", True),
                              ("none_grow_arena", "none", True)):
        if grow:
            os.environ.pop("CEL_NO_GROW", None)
        else:
            os.environ["CEL_NO_GROW"] = "1"
        if label == "none_grow_arena":
            os.environ["CEL_NO_VMM"] = "1"
        else:
            os.environ.pop("CEL_NO_VMM", None)
        rt = cel.Runtime(1, lookahead=mode, arena_bytes=4 << 30)
        prog = P.rsim(W, T)
        rt.buffer_create(2, [T, W], 4)
        descs = [cel.task_desc(op[1]) for op in prog["ops"] if op[0] == "task"]
        rt.profile_enable(True)
        dt = timed(rt, lambda: [rt.submit_desc(d[0]) for d in descs])
        prof = rt.profile_read()
        st = rt.stats()
        rt.shutdown()
        cm = prof.get("copy", (0.0, 0))
        km = prof.get("rsim_row", (0.0, 0))[0] / 1e3
        kbytes = sum(t * W * 4 for t in range(1, T)) + (T - 1) * W * 4
        res[label] = {"seconds": dt, "resize_copies_elided": st["copies_elided"], "steps_per_s": T / dt, "alloc": st["n_alloc"], "flushes": st["flushes"],
                     "vmm_maps": st["vmm_maps"],
                     "resize_copies": st["copies_resize"], "resize_bytes": st["bytes_resize"],
                     "resize_copy_GBps": (2 * st["bytes_resize"] / (cm[0] / 1e3) / 1e9) if cm[0] else None,
                     "kernel_GBps": kbytes / km / 1e9 if km else None, "profile_ms": {k: v[0] for k, v in prof.items()}}
    os.environ.pop("CEL_NO_GROW", None)
    os.environ.pop("CEL_NO_VMM", None)
    res["speedup_auto_vs_none"] = res["none"]["seconds"] / res["auto"]["seconds"]
    res["speedup_auto_vs_none_grow"] = res["none_grow"]["seconds"] / res["auto"]["seconds"]
    return res


def c5(steps=40, n=1024):
    """C5 at G=1: wall-clock steps/s between two epochs (no profiling in the
    timed window; per-launch profile events add ~4% to a 1.4 ms kernel)."""
    G = 1
    rt = cel.Runtime(G, arena_bytes=int(2 * n ** 3 * 4 * 1.05) + (512 << 20))
    prog = P.jacobi3d(n, 2)
    rt.buffer_create(3, [n, n, n], 4)
    rt.buffer_create(3, [n, n, n], 4)
    rt.task_submit(prog["ops"][0][1])
    d = [cel.task_desc(P.jacobi_step(n, k)[1]) for k in (0, 1)]
    for k in range(4):
        rt.submit_desc(d[k % 2][0])
    dt = timed(rt, lambda: [rt.submit_desc(d[k % 2][0]) for k in range(steps)])
    rt.shutdown()
    alg = 8.0 * n ** 3
    ach = alg * steps / dt / 1e9
    return {"steps_per_s": steps / dt, "kernel": "jacobi7_tma (TMA tensor-map plane tiles)",
            "roofline": {"bound": "hbm", "achieved": ach, "peak": HBM, "unit": "GB/s", "frac": ach / HBM,
                         "alg_bytes_per_launch": alg, "basis": "wall-clock per step (one launch per step)"},
            "devices": G}


def copy_sweep():
    out = {"impl": os.environ.get("CEL_COPY", "lsu")}
    # measure the copies themselves: in-place growth would turn these resizes
    # into no-ops (the arena range after the allocation is free)
    grow = os.environ.get("CEL_NO_GROW")
    os.environ["CEL_NO_GROW"] = "1"
    # (a) 1 GiB contiguous resize copy: write [0, 2^28), then a task needs [0, 2^28 + 1)
    n = 1 << 28
    for reps in range(2):          # the first run pays lazy module loading; the second is reported
        rt = cel.Runtime(1, lookahead="none", arena_bytes=3 << 30)
        rt.buffer_create(1, [n + 1], 4)
        rt.task_submit({"dims": 1, "range": ([0], [n]), "kernel": "fill_const", "params": {"value": 1.0},
                        "accesses": [(0, "write", ("one_to_one",))]})
        rt.wait()
        rt.profile_enable(True)
        dt = timed(rt, lambda: rt.task_submit({"dims": 1, "range": ([0], [n + 1]), "kernel": "fill_const",
                                               "params": {"value": 2.0},
                                               "accesses": [(0, "read_write", ("one_to_one",))]}))
        prof = rt.profile_read()
        rt.shutdown()
        ms = prof["copy"][0]
        out["resize_1GiB"] = {"payload_bytes": 4 * n, "ms": ms, "GBps_rw": 2 * 4 * n / (ms / 1e3) / 1e9,
                              "frac_hbm": 2 * 4 * n / (ms / 1e3) / 1e9 / HBM}
    # (b) strided 2-D resize: 8192 rows x 16 KiB out of a 16 KiB-pitch into a 16 KiB+4 B pitch allocation
    R, Cc = 8192, 4096
    rt = cel.Runtime(1, lookahead="none", arena_bytes=2 << 30)
    rt.buffer_create(2, [R, 16384], 4)
    rt.task_submit({"dims": 2, "range": ([0, 0], [R, Cc]), "kernel": "fill_const", "params": {"value": 1.0},
                    "accesses": [(0, "write", ("one_to_one",))]})
    rt.wait()
    rt.profile_enable(True)
    timed(rt, lambda: rt.task_submit({"dims": 2, "range": ([0, 0], [R, Cc + 1]), "kernel": "fill_const",
                                      "params": {"value": 2.0}, "accesses": [(0, "read_write", ("one_to_one",))]}))
    prof = rt.profile_read()
    rt.shutdown()
    ms = prof["copy"][0]
    out["resize_2d_8192x16KiB"] = {"payload_bytes": R * Cc * 4, "ms": ms,
                                   "GBps_rw": 2 * R * Cc * 4 / (ms / 1e3) / 1e9,
                                   "frac_hbm": 2 * R * Cc * 4 / (ms / 1e3) / 1e9 / HBM}
    # (c) peer pushes over NVLink: every device pulls the other's half (an 'all' read)
    if torch.cuda.device_count() >= 2:
        for mib in (16, 256, 1024):
            N = mib * (1 << 20) // 16
            # collective=False: this row measures the peer-push copy kernel (the
            # all-gather set would otherwise run as NCCL, measured by c3 / configs)
            rt = cel.Runtime(2, cuda_devices=[0, 1], arena_bytes=3 << 30, collective=False)
            rt.buffer_create(1, [N], 16)
            rt.buffer_create(1, [N], 16)
            rt.task_submit({"dims": 1, "range": ([0], [N]), "kernel": "fill_const", "params": {"value": 1.0},
                            "accesses": [(0, "write", ("one_to_one",))]})
            rt.wait()
            rt.profile_enable(True)
            timed(rt, lambda: rt.task_submit({"dims": 1, "range": ([0], [N]), "kernel": "fill_const",
                                              "params": {"value": 2.0},
                                              "accesses": [(0, "read", ("all",)), (1, "write", ("one_to_one",))]}))
            prof = rt.profile_read()
            rt.shutdown()
            ms, cnt = prof["copy_peer"]
            half = N * 16 // 2
            out["peer_push_%dMiB" % mib] = {"payload_bytes_per_copy": half, "copies": cnt, "ms_total": ms,
                                            "GBps_per_direction": half / (ms / cnt / 1e3) / 1e9,
                                            "frac_nvlink_nominal": half / (ms / cnt / 1e3) / 1e9 / NVLINK_NOMINAL,
                                            "frac_nvlink_measured_ref": half / (ms / cnt / 1e3) / 1e9 / NVLINK_MEASURED_REF}
    if grow is None:
        os.environ.pop("CEL_NO_GROW", None)
    else:
        os.environ["CEL_NO_GROW"] = grow
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="c1,c3,c3fast,c4,c5,copy")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    res = {"gpu": torch.cuda.get_device_name(0), "gpus": torch.cuda.device_count(), "hbm_peak_gbs": HBM,
           "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())}
    fns = {"c1": c1, "c3": c3, "c3fast": c3fast, "c4": c4, "c5": c5, "copy": copy_sweep}
    for k in args.only.split(","):
        t0 = time.time()
        res[k] = fns[k]()
        res[k]["wall_s"] = time.time() - t0
        print(k, json.dumps(res[k]), flush=True)
    if args.out:
        json.dump(res, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
