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
    """Clock / throttle sampling DURING the timed region (the recipe's clocks
    line): an NVML thread samples every millisecond (the timed region of a
    short run is only milliseconds long), falling back to `nvidia-smi -lms`."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown", 0x4: "sw_power_cap",
               0x80: "hw_power_brake_slowdown"}

    def __init__(self, gpu):
        import threading
        self.rows = []
        self.p = None
        self.stop_ev = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(vis.split(",")[gpu]) if vis and vis.split(",")[gpu].strip().isdigit() else gpu
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.sample()
            self.t = threading.Thread(target=self.loop, daemon=True)
            self.t.start()
        except Exception:
            self.nv = None
            self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
            q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
            try:
                self.p = subprocess.Popen(["nvidia-smi", "-i", str(gpu), "--query-gpu=" + q,
                                           "--format=csv,noheader,nounits", "-lms", "100"],
                                          stdout=self.f, stderr=subprocess.DEVNULL)
            except Exception:
                self.p = None

    def sample(self):
        nv = self.nv
        try:
            r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        except Exception:
            r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
        self.rows.append((float(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)), float(self.max_mhz),
                          [v for k, v in self.REASONS.items() if r & k]))

    def loop(self):
        while not self.stop_ev.wait(0.001):
            self.sample()

    def stop(self):
        if self.nv is not None:
            self.sample()
            self.stop_ev.set()
            self.t.join()
            rows = self.rows
            how = "nvml, 1 ms"
        else:
            if self.p is None:
                return None
            self.p.terminate()
            try:
                self.p.wait(timeout=5)
            except Exception:
                self.p.kill()
            self.f.flush()
            rows = []
            names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
            for line in open(self.f.name):
                parts = [x.strip() for x in line.split(",")]
                if len(parts) < 9:
                    continue
                try:
                    rows.append((float(parts[1]), float(parts[2]),
                                 [names[i] for i, v in enumerate(parts[5:9]) if v.lower() == "active"]))
                except ValueError:
                    continue
            os.unlink(self.f.name)
            how = "nvidia-smi, 100 ms"
        if not rows:
            return None
        sm = sorted(r[0] for r in rows)
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": max(r[1] for r in rows),
                "reasons": sorted({x for r in rows for x in r[2]}), "samples": len(rows), "sampler": how}


def oracle_wave_fields(rows, seed=2):
    """u = up = the input recipe's init(seed, .) (the WaveSim workload's fill
    tasks) over `rows` full-width rows of the 16384^2 field plus one halo row
    on each side when rows < 16384, as the oracle's accessors; returns them
    and the box of rows a step writes."""
    import numpy as np
    from oracle import geometry as g
    from oracle.kernels import Acc, init_value
    lo, hi = (0, N_FIELD) if rows >= N_FIELD else (0, rows + 2)
    idx = np.arange(lo * N_FIELD, hi * N_FIELD, dtype=np.uint64)
    f = np.asarray(init_value(seed, idx), dtype=np.float32).reshape(hi - lo, N_FIELD, 1, 1).view(np.uint32)
    ext = g.box([0, 0], [N_FIELD, N_FIELD])
    box = g.box([lo, 0], [hi, N_FIELD])
    wbox = box if rows >= N_FIELD else g.box([1, 0], [rows + 1, N_FIELD])
    return Acc(f.copy(), box, ext), Acc(f, box, ext), wbox


def oracle_wave_step(U, UP, wbox, k):
    """One WaveSim step of the oracle (oracle.kernels.k_wave5, NumPy float32,
    one core) over the rows of wbox."""
    from oracle.kernels import k_wave5
    k_wave5({}, [wbox, wbox], [U, UP] if k % 2 == 0 else [UP, U])


def cpu_baseline(budget_s=15.0, max_steps=3):
    """The oracle as it stands, timed on this host: WaveSim steps of the full
    16384^2 field through the oracle's wave5 kernel (G = 1: the IDAG is one
    kernel instruction per step, its generation is negligible), repeated until
    budget_s or max_steps -- measured at full size, not extrapolated."""
    import time as _t
    U, UP, box = oracle_wave_fields(N_FIELD)
    k, dt = 0, 0.0
    while k < max_steps and (k == 0 or dt < budget_s):
        t0 = _t.perf_counter()
        oracle_wave_step(U, UP, box, k)
        dt += _t.perf_counter() - t0
        k += 1
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    return {"value": k / dt, "unit": "steps/s", "cores": 1, "kind": "oracle",
            "sample": "%d full-size steps of WaveSim 16384^2 f32 (oracle.kernels.k_wave5, NumPy, one thread; host "
                      "has %d cores), measured" % (k, cores),
            "seconds": dt}


def run_reference(args):
    """--impl reference: the oracle, as it stands, on this arm's metric.  Each
    timed step is one WaveSim step through the oracle's wave5 kernel over R
    full-width rows: R = 16384 (the whole field, measured) when K full steps
    fit in about 100 s of CPU, else the largest slab that does, the line then
    scaled by rows and saying so.  Warm-up steps run on a 64-row slab."""
    rank, world, _ = env_rank()
    if rank != 0:
        return
    import time as _t
    Uw, UPw, bw = oracle_wave_fields(64)
    for k in range(args.warmup):
        oracle_wave_step(Uw, UPw, bw, k)
    t0 = _t.perf_counter()
    oracle_wave_step(Uw, UPw, bw, 0)
    per_row = (_t.perf_counter() - t0) / 64
    R = int(min(N_FIELD, max(64, 100.0 / max(1, args.steps) / max(per_row, 1e-9))))
    U, UP, box = oracle_wave_fields(R)
    t0 = _t.perf_counter()
    for k in range(args.steps):
        oracle_wave_step(U, UP, box, k)
    dt = _t.perf_counter() - t0
    val = args.steps * (R / N_FIELD) / dt
    sample = ("oracle wave5 kernel (NumPy, one thread), %d steps of the full 16384^2 field, measured" % args.steps
              if R == N_FIELD else
              "oracle wave5 kernel (NumPy, one thread), %d steps over %d of 16384 rows each, scaled by rows "
              "(full-size steps would not fit the run's time budget)" % (args.steps, R))
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "steps/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 / val,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": arm_config(args.gpus, world),
            "cpu_baseline": {"value": val, "unit": "steps/s", "cores": 1, "kind": "oracle", "sample": sample},
            "e2e": {"value": val, "unit": "steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def copy_block(cel, P, peak):
    """The coherence-copy half of BASELINE.json's metric ("coherence copy GB/s
    vs HBM peak"), through the product path on this GPU: resize copies (alloc
    -> copy -> free) of 1 GiB contiguous and 8192 x 16 KiB strided, and
    halo-shaped coherence copies between virtual devices (WaveSim 64 KiB rows;
    3-D faces: 2 MiB z-faces, 256 x 4 KiB strided y-faces, corner lines).
    Device time per copy launch from the library's CUDA-event profile; bytes
    are read + write of HBM (2 x payload); resized data byte-checked."""
    import numpy as np
    out = {}
    saved = os.environ.get("CEL_NO_GROW")
    os.environ["CEL_NO_GROW"] = "1"            # measure real resize copies, not in-place growth

    def resize_case(name, ext, written, fixed, samples, copy_impl=None, reps=2):
        for _ in range(reps):                  # the first run pays lazy module loading: report the last
            resize_once(name, ext, written, fixed, samples, copy_impl)

    def resize_once(name, ext, written, fixed, samples, copy_impl):
        prev = os.environ.get("CEL_COPY")
        if copy_impl:
            os.environ["CEL_COPY"] = copy_impl
        rt = cel.Runtime(1, lookahead="none", arena_bytes=3 << 30)
        if copy_impl:
            if prev is None:
                os.environ.pop("CEL_COPY", None)
            else:
                os.environ["CEL_COPY"] = prev
        dims = len(ext)
        rt.buffer_create(dims, ext, 4)
        rt.task_submit({"dims": dims, "range": ([0] * dims, list(written)), "kernel": "fill_hash",
                        "params": {"seed": 11}, "accesses": [(0, "write", ("one_to_one",))]})
        rt.wait()
        rt.profile_enable(True)
        # a 1-item task writing a box that overlaps the live allocation's end:
        # R9 merges them, i.e. one resize copy of the whole written part
        rt.task_submit({"dims": 1, "range": ([0], [1]), "kernel": "fill_const", "params": {"value": 2.0},
                        "accesses": [(0, "write", ("fixed", fixed))]})
        rt.wait()
        prof = rt.profile_read()
        st = rt.stats()
        ok = True
        for lo, hi in samples:
            got = rt.buffer_read(0, (lo, hi)).view(np.float32).reshape(-1)
            grid = np.indices([h - l for l, h in zip(lo, hi)]).reshape(len(lo), -1)
            lin = np.zeros(grid.shape[1], dtype=np.uint64)
            for d in range(dims):
                lin = lin * np.uint64(ext[d]) + (grid[d] + lo[d]).astype(np.uint64)
            ok = ok and np.array_equal(got.view(np.uint32), P.init_values(11, lin).view(np.uint32))
        rt.shutdown()
        ms, cnt = prof.get("copy", (0.0, 0))
        payload = st["bytes_resize"]
        gbs = 2 * payload / (ms / 1e3) / 1e9 if ms else None
        out[name] = {"payload_bytes": payload, "copies": st["copies_resize"], "launches": cnt, "ms": ms,
                     "GBps_hbm_rw": gbs, "frac_hbm": gbs / peak if gbs else None, "bytes_ok": bool(ok),
                     "kernel": "copy_kernel_tmap (TMA tensor maps)" if st["tma_copy_launches"] else "copy_kernel (LSU)"}

    n = 1 << 28
    resize_case("resize_1GiB", [n + 1], [n], ([n - 1], [n + 1]),
                [([0], [1 << 20]), ([n // 2], [n // 2 + (1 << 20)]), ([n - (1 << 20)], [n - 1])])
    R, C = 8192, 4096
    resize_case("resize_2d_8192x16KiB", [R, 16384], [R, C], ([0, C - 1], [R, C + 1]),
                [([0, 0], [64, C - 1]), ([R // 2, 0], [R // 2 + 64, C - 1]), ([R - 64, 0], [R, C - 1])])
    resize_case("resize_2d_8192x16KiB_tma", [R, 16384], [R, C], ([0, C - 1], [R, C + 1]),
                [([0, 0], [64, C - 1]), ([R // 2, 0], [R // 2 + 64, C - 1]), ([R - 64, 0], [R, C - 1])], "tma")
    # 3-D: 256 planes x 64 rows x 4 KiB at a 256 KiB plane pitch into a 260 KiB one
    resize_case("resize_3d_256x64x4KiB", [256, 80, 1024], [256, 64, 1024], ([0, 63, 0], [256, 65, 1024]),
                [([0, 0, 0], [2, 63, 1024]), ([255, 0, 0], [256, 63, 1024])])
    resize_case("resize_3d_256x64x4KiB_tma", [256, 80, 1024], [256, 64, 1024], ([0, 63, 0], [256, 65, 1024]),
                [([0, 0, 0], [2, 63, 1024]), ([255, 0, 0], [256, 63, 1024])], "tma")
    if saved is None:
        os.environ.pop("CEL_NO_GROW", None)
    else:
        os.environ["CEL_NO_GROW"] = saved

    def halo_case(name, G, ext, descs_of, init, steps):
        rt = cel.Runtime(G, cuda_devices=[0] * G, arena_bytes=int(2 * np.prod(ext) * 4 / G * 1.3) + (256 << 20))
        rt.buffer_create(len(ext), ext, 4)
        rt.buffer_create(len(ext), ext, 4)
        for op in init:
            rt.task_submit(op[1])
        descs = [cel.task_desc(d[1]) for d in descs_of]
        for k in range(4):
            rt.submit_desc(descs[k % 2][0])
        rt.wait()
        st0 = rt.stats()
        rt.profile_enable(True)
        for k in range(steps):
            rt.submit_desc(descs[k % 2][0])
        rt.wait()
        prof = rt.profile_read()
        st1 = rt.stats()
        rt.shutdown()
        ms, cnt = prof.get("copy", (0.0, 0))
        payload = st1["bytes_coherence"] - st0["bytes_coherence"]
        copies = st1["copies_coherence"] - st0["copies_coherence"]
        gbs = 2 * payload / (ms / 1e3) / 1e9 if ms else None
        out[name] = {"devices": "%d virtual devices on one GPU" % G, "in_situ": "timed while the stencil runs "
                     "(latency-bound: a launch per copy instruction)", "copies": copies, "launches": cnt,
                     "payload_bytes": payload, "us_per_copy": ms * 1e3 / cnt if cnt else None,
                     "GBps_hbm_rw": gbs, "frac_hbm": gbs / peak if gbs else None}

    nf = N_FIELD
    halo_case("halo_rows_64KiB", 2, [nf, nf], [P.wavesim_step(nf, k) for k in (0, 1)], P.wavesim_init(nf), 200)
    nz = 512
    jac = P.jacobi3d(1024, 2)
    jac_init = [("task", dict(jac["ops"][0][1], range=([0, 0, 0], [nz, 1024, 1024])))]
    steps = [("task", dict(P.jacobi_step(1024, k)[1], range=([0, 0, 0], [nz, 1024, 1024]))) for k in (0, 1)]
    halo_case("halo_3d_faces_2x2", 4, [nz, 1024, 1024], steps, jac_init, 40)
    return out


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
    ap.add_argument("--no-copy", action="store_true")
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
    halo_fused = st1.get("halo_fused", 0) - st0.get("halo_fused", 0)
    if halo_fused:
        # halo exchange fused into the stencil (exec_halo.cu): one launch per
        # step covers the whole chunk, the boundary rows included
        interior_rows = rows_here
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
    copies = None
    if G == 1 and world == 1 and not args.no_copy:
        copies = copy_block(cel, P, peak)
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
                     "kernel": "wave5_halo" if halo_fused else "wave5_vec", "alg_bytes_per_launch": alg_bytes,
                     "avg_launch_ms": avg_s * 1e3 if wcnt else None,
                     "shell_ms_per_step": shell_ms / args.steps,
                     "peak_source": peak_kind + " hbm_gbs",
                     "kernel_share_of_step": kernel_share},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "copy": copies,
        "gpu_launches": launches,
        "halo_fused_per_step": halo_fused / args.steps,
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
