"""Benchmark: WaveSim 16384^2 fp32 steps/s through the coherence path (C-ABI).

Contract (see task statement / DESIGN.md §6):
  python bench.py --gpus N --steps K --warmup W            (N=1 runs directly;
  N>1 is launched by torchrun, one process per GPU, RANK/WORLD_SIZE from env)
prints ONE JSON line on rank 0.  `value` is whole-job WaveSim steps/s of the
fixed 16384^2 problem split over the N GPUs (strong scaling), timed with CUDA
events between two epochs, max over ranks.  `e2e` is the same metric through
the public API with host buffers (H2D of the initial fields and D2H of the
result inside the timed region).  `roofline` is the WaveSim kernel's
algorithmic bytes / its CUDA-event launch time vs the measured HBM peak;
`cpu_baseline` is the CPU oracle on a bounded sample (rank 0, N=1 only).
`--impl reference` times the oracle itself on the same metric.
"""

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_FIELD = 16384
METRIC = "WaveSim steps/s (16384^2 fp32, 1-D row split, halo coherence copies)"


def arm_config(G, world, n=N_FIELD):
    """The `config` both arms (ours and --impl reference) report."""
    return {"workload": "wavesim_%dx%d_f32" % (n, n), "n_devices": G, "split": "1d rows", "lookahead": "auto",
            "processes": world,
            "l2": "inputs larger than L2 (u+up = %.2f GiB per GPU vs 126 MB L2)" % (2 * n * n * 4 / G / 2 ** 30)}
ALG_BYTES_PER_CELL = 12        # wave5: read u, read up, write up (4 B each)
PROF_STRIDE = 8


def env_rank():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get("hbm_gbs", 6650.0), "measured"
    return 6650.0, "fallback"


class Clocks:
    """nvidia-smi sampling during the timed region (the recipe's clocks line)."""

    def __init__(self, gpu):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(gpu), "--query-gpu=" + q, "--format=csv,noheader,nounits",
                                       "-lms", "100"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        self.f.flush()
        rows = []
        for line in open(self.f.name):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                rows.append((float(parts[1]), float(parts[2]), parts[5:9]))
            except ValueError:
                continue
        os.unlink(self.f.name)
        if not rows:
            return None
        sm = sorted(r[0] for r in rows)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i, v in enumerate(r[2]) if v.lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": max(r[1] for r in rows), "reasons": reasons,
                "samples": len(rows)}


def cpu_baseline(budget_s=12.0, max_reps=8):
    """The oracle, as it stands, on a bounded sample of the WaveSim workload:
    16384 columns x R rows, IDAG generation + byte simulation, one process,
    repeated until about budget_s of CPU work.  Scaled to full 16384^2
    steps/s by rows."""
    import numpy as np  # noqa: F401
    from oracle.scheduler import Runtime as OracleRuntime, run_program
    from oracle.simulate import simulate
    from workloads import programs as P
    rows, steps = 1024, 3
    reps, dt = 0, 0.0
    while reps < max_reps and (reps == 0 or dt < budget_s):
        t0 = time.perf_counter()
        prog = P.wavesim(N_FIELD, steps, rows=rows)
        prog["ops"] = [op for op in prog["ops"] if op[0] != "read"] + [("read", 1, P.full([rows, N_FIELD]))]
        o = OracleRuntime(1)
        run_program(o, prog)
        simulate(o)
        dt += time.perf_counter() - t0
        reps += 1
    full_steps = reps * steps * rows / N_FIELD
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    return {"value": full_steps / dt, "unit": "steps/s", "cores": 1, "kind": "oracle",
            "sample": "%d x (WaveSim %d rows x %d cols, %d steps incl. 2 fills), oracle IDAG + NumPy byte "
                      "simulation, scaled by rows to 16384^2 steps (host has %d cores; NumPy elementwise is "
                      "single-threaded)" % (reps, rows, N_FIELD, steps, cores),
            "seconds": dt}


def run_reference(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return
    import numpy as np
    from oracle import geometry as g
    from oracle.kernels import Acc, k_wave5
    # each "step" is a bounded sample: one wave5 step over R rows of the 16384^2
    # field through the oracle kernel (pure NumPy, 1 core), scaled by rows
    # bounded: ~1 ms of NumPy per row, keep the whole run around a minute
    R = int(max(8, min(512, 60000 // max(1, args.steps + args.warmup))))
    ext = g.box([0, 0], [N_FIELD, N_FIELD])
    rng = np.random.default_rng(2)
    u = rng.uniform(-1, 1, (R + 2, N_FIELD, 1, 1)).astype(np.float32).view(np.uint32)
    up = rng.uniform(-1, 1, (R + 2, N_FIELD, 1, 1)).astype(np.float32).view(np.uint32)
    ubox = g.box([0, 0], [R + 2, N_FIELD])
    wbox = g.box([1, 0], [R + 1, N_FIELD])
    U, UP = Acc(u, ubox, ext), Acc(up, ubox, ext)
    for _ in range(args.warmup):
        k_wave5({}, [ubox, wbox], [U, UP])
    t0 = time.perf_counter()
    for k in range(args.steps):
        if k % 2 == 0:
            k_wave5({}, [ubox, wbox], [U, UP])
        else:
            k_wave5({}, [ubox, wbox], [UP, U])
    dt = time.perf_counter() - t0
    full = args.steps * R / N_FIELD
    val = full / dt
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "steps/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 / val,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": arm_config(args.gpus, world),
            "cpu_baseline": {"value": val, "unit": "steps/s", "cores": 1, "kind": "oracle",
                             "sample": "oracle wave5 kernel on %d of 16384 rows per step, scaled by rows" % R},
            "e2e": {"value": val, "unit": "steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def gpu_of(v):
    """Physical GPU of virtual device / rank v.  CEL_BENCH_GPUS=k folds the
    ranks onto k GPUs (several processes per GPU): a functional rehearsal of
    N > k runs on a smaller box, not a performance measurement."""
    k = int(os.environ.get("CEL_BENCH_GPUS", "0") or 0)
    return v % k if k > 0 else v


def make_runtime(cel, G, rank, world, dist, arena, **kw):
    devs = [gpu_of(v) for v in range(G)]
    if world > 1:
        rt = cel.Runtime(G, cuda_devices=devs, arena_bytes=arena, rank=rank, world=world, **kw)
        blob = rt.ipc_export()
        blobs = [None] * world
        dist.all_gather_object(blobs, blob)
        for r, b in enumerate(blobs):
            if r != rank:
                rt.ipc_import(r, b)
        dist.barrier()
        return rt
    return cel.Runtime(G, cuda_devices=devs, arena_bytes=arena, **kw)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=N_FIELD)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        run_reference(args)
        return

    import numpy as np
    import torch
    from paper_2503_10516_b200 import cel
    from workloads import programs as P

    rank, world, local = env_rank()
    G = args.gpus
    if world > 1 and world != G:
        raise SystemExit("--gpus must equal WORLD_SIZE under torchrun")
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")
    torch.cuda.set_device(gpu_of(local) if world > 1 else 0)
    n = args.n
    arena = int(2 * (n // G + 2) * n * 4 * 1.05) + (512 << 20)

    rt = make_runtime(cel, G, rank, world, dist, arena)
    u = rt.buffer_create(2, [n, n], 4)
    up = rt.buffer_create(2, [n, n], 4)
    for op in P.wavesim_init(n):
        rt.task_submit(op[1])
    descs = [cel.task_desc(P.wavesim_step(n, k)[1]) for k in (0, 1)]

    def steps(k0, k):
        for s in range(k0, k0 + k):
            rt.submit_desc(descs[s % 2][0])

    steps(0, args.warmup)
    rt.wait()
    # ---- timed region: K steps between two epochs
    st0 = rt.stats()
    if not os.environ.get("CEL_BENCH_NOPROF"):
        # CUDA events around every 8th launch of each kind: the average launch
        # duration of the timed region at 1/8 of the event overhead (timing
        # every launch cost 6.7% of the step at 4 GPUs)
        rt.profile_enable(True, stride=PROF_STRIDE)
    clk = Clocks(local) if rank == 0 else None
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    sh0 = rt.stats()
    th0 = time.perf_counter()
    # host cost per step: measured over the first steps, before the executor's
    # in-flight cap (2048 events per stream) starts pacing the host to the GPU
    kh = min(args.steps, 300)
    steps(args.warmup, kh)
    th1 = time.perf_counter()
    sh1 = rt.stats()
    steps(args.warmup + kh, args.steps - kh)
    rt.wait()
    ev1.record()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    ms = ev0.elapsed_time(ev1)
    clocks = clk.stop() if clk else None
    prof = rt.profile_read()
    rt.profile_enable(False)
    st1 = rt.stats()
    if dist:
        t = torch.tensor([ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    launches = st1["kernel_launches"] - st0["kernel_launches"]
    rt.shutdown()

    # ---- roofline of the dominant kernel (wave5 on this rank's chunk)
    peak, peak_kind = measured_peaks()
    wms, wcnt = prof.get("wave5", (0.0, 0))
    rows_here = n // G + (1 if (rank if world > 1 else 0) < n % G else 0)
    alg_bytes = ALG_BYTES_PER_CELL * rows_here * n
    # one wave5 instruction per device per step; with halo overlap it runs as a
    # shell launch (profiled separately) + an interior launch: the roofline is
    # the interior launch, over the interior's algorithmic bytes
    inst_per_rank = args.steps * (G if world == 1 else 1)
    shell_ms, shell_cnt = prof.get("shell", (0.0, 0))
    shell_ms *= PROF_STRIDE                  # sampled: every PROF_STRIDE-th shell launch timed
    border_rows = (0 if (world > 1 and rank == 0) or (world == 1 and G == 1) else 1) + \
                  (0 if (world > 1 and rank == world - 1) or (world == 1 and G == 1) else 1)
    if world == 1 and G > 1:
        border_rows = 2 * (G - 1) / G
    interior_rows = rows_here - border_rows
    avg_s = (wms / wcnt) / 1e3 if wcnt else float("nan")         # sampled launches: unbiased average
    alg_bytes = ALG_BYTES_PER_CELL * interior_rows * n
    achieved = alg_bytes / avg_s / 1e9 if wcnt else None
    traffic = None
    tp = os.path.join(ROOT, "profiles", "wave5_traffic.json")
    if os.path.exists(tp):
        traffic = json.load(open(tp)).get("bytes_per_cell") * rows_here * n
    step_ms = ms / args.steps
    value = 1e3 / step_ms
    kernel_share = (avg_s * 1e3 * inst_per_rank / (ms * (G if world == 1 else 1))) if ms and wcnt else None

    # ---- e2e: host buffers in, result out, through the public API
    e2e = None
    if not args.no_e2e:
        ke = max(args.steps, 50)
        rng = np.random.default_rng(2)
        host_u = torch.from_numpy(rng.uniform(-1, 1, (n, n)).astype(np.float32)).pin_memory().numpy()
        host_up = torch.from_numpy(host_u.copy()).pin_memory().numpy()
        res = torch.empty((n, n), dtype=torch.float32).pin_memory().numpy()
        # the runtime (arena reservation, IPC handle exchange) is set up once,
        # before the timed region: the user's session, not part of a run
        rt2 = make_runtime(cel, G, rank, world, dist, arena)
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        b0 = rt2.buffer_create(2, [n, n], 4, host_init=host_u, borrow=True)
        b1 = rt2.buffer_create(2, [n, n], 4, host_init=host_up, borrow=True)
        d2 = [cel.task_desc(P.wavesim_step(n, k)[1]) for k in (0, 1)]
        for s in range(ke):
            rt2.submit_desc(d2[s % 2][0])
        last = b1 if ke % 2 == 1 else b0
        rt2.buffer_read(last, ([0, 0], [n, n]), out=res.reshape(n, n, 1, 1).view(np.uint32))
        t1 = time.perf_counter()
        rt2.shutdown()
        el = t1 - t0
        if dist:
            t = torch.tensor([el], dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            el = float(t.item())
        e2e = {"value": ke / el, "unit": "steps/s", "h2d_bytes_per_step": int(2 * n * n * 4 / G / ke),
               "d2h_bytes_per_step": int(n * n * 4 / G / ke), "steps": ke,
               "includes": "H2D of both 16384^2 fields from pinned host memory (borrowed, "
                            "DMA) + %d steps + D2H readback of the result into pinned memory" % ke}

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return
    cpu = None
    if G == 1 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline()
    line = {
        "metric": METRIC,
        "value": value, "unit": "steps/s", "n_gpus": G, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": step_ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic",
        "config": arm_config(G, world, n),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                     "kernel": "wave5_vec", "alg_bytes_per_launch": alg_bytes,
                     "avg_launch_ms": avg_s * 1e3 if wcnt else None,
                     "shell_ms_per_step": shell_ms / args.steps,
                     "peak_source": peak_kind + " hbm_gbs",
                     "kernel_share_of_step": kernel_share},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": launches,
        "host_submit_us_per_step": (th1 - th0) / kh * 1e6,
        "host_us_per_step_by_part": {k[8:] if k.startswith("exec_ns_") else k: (sh1[k] - sh0[k]) / kh / 1e3
                                     for k in ("exec_ns_copy", "exec_ns_kernel", "exec_ns_alloc", "exec_ns_free",
                                               "exec_ns_horizon", "signal_ns", "remote_wait_ns")},
        "clocks": clocks,
        "profile_ms": {k: {"ms": v[0], "launches": v[1]} for k, v in prof.items()},
        "profile_stride": PROF_STRIDE,
    }
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
