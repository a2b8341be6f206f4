"""GPU parity: the CUDA path (C-ABI, sm_100a kernels) against the CPU oracle.

Bit-exact for every readback (integer probes and fp32 under -fmad=false, R16)
and record-for-record equality of the instruction logs.  Several virtual
devices may share one physical GPU (the multi-device logic — separate
allocations, streams, d2d copies — is exercised on one B200); with >= 2 GPUs
the same programs also run across physical devices (peer copies over NVLink).
"""

import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import geometry as g  # noqa: E402
from oracle.kernels import Acc, init_value, k_wave5, nbody_accel_one  # noqa: E402
from oracle.scheduler import Runtime as OracleRuntime  # noqa: E402
from workloads.driver import run_program  # noqa: E402
from oracle.simulate import simulate  # noqa: E402
from workloads import programs as P  # noqa: E402

LOG = "/tmp/cel_gpu_log.jsonl"


@pytest.fixture(scope="module")
def cel():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import __graft_entry__
    __graft_entry__.build()
    from paper_2503_10516_b200 import cel as c
    return c


def run_both(cel, prog, G, mode="auto", devices=None, arena=256 << 20, step=4):
    devices = devices if devices is not None else [0] * G
    rt = cel.Runtime(G, cuda_devices=devices, lookahead=mode, arena_bytes=arena, instr_log_path=LOG,
                     horizon_step=step)
    close = rt.shutdown

    def shutdown():                  # keep the final executor statistics for the caller
        if rt.h is not None:
            rt.final_stats = rt.stats()
        close()
    rt.shutdown = shutdown
    got = [r[1] for r in run_program(rt, prog) if r[0] == "read"]
    o = OracleRuntime(G, lookahead=mode, horizon_step=step)
    run_program(o, prog)
    exp = simulate(o)
    log = [json.loads(line) for line in open(LOG)]
    assert log == o.log, "instruction log differs from the oracle"
    for k, arr in enumerate(got):
        e = exp[k]
        defined = e != np.uint32(0x7FC00BAD)      # never-written elements are not compared (R6)
        if not np.array_equal(arr[defined], e[defined]):
            bad = np.argwhere((arr != e) & defined)
            raise AssertionError("readback %d: %d mismatches, first at %s" % (k, len(bad), bad[:3].tolist()))
    return rt


def test_smoke(cel):
    import __graft_entry__
    __graft_entry__.smoke()


@pytest.mark.parametrize("G", [1, 2, 3, 4])
def test_random_programs(cel, G):
    for s in range(12):
        prog = P.random_program(9000 + 17 * G + s)
        for mode in ("none", "auto"):
            run_both(cel, prog, G, mode, arena=32 << 20, step=2 + s % 3)


@pytest.mark.parametrize("G", [1, 2, 4])
@pytest.mark.parametrize("mode", ["none", "auto"])
def test_c1_chain(cel, G, mode):
    run_both(cel, P.c1_chain(4096), G, mode)


@pytest.mark.parametrize("G,rows,cols", [(1, 64, 512), (2, 300, 1040), (3, 257, 2048), (4, 130, 516), (2, 77, 101)])
def test_wavesim_ragged(cel, G, rows, cols):
    # several strips and CTAs, ragged tails; cols=101 takes the scalar kernel
    run_both(cel, P.wavesim(cols, 9, rows=rows), G)


@pytest.mark.parametrize("G", [1, 2, 4, 8])
def test_jacobi3d(cel, G):
    run_both(cel, P.jacobi3d(36, 5), G)


def test_jacobi3d_ragged(cel):
    prog = P.jacobi3d(20, 3)
    run_both(cel, prog, 6)


@pytest.mark.parametrize("G", [1, 3])
def test_nbody(cel, G):
    run_both(cel, P.nbody(1000, 2), G)
    run_both(cel, P.nbody(300, 2, host_init=True), G)


@pytest.mark.parametrize("G,mode", [(1, "auto"), (2, "auto"), (2, "none"), (4, "none"), (3, "infinite")])
def test_rsim(cel, G, mode):
    run_both(cel, P.rsim(1000, 24), G, mode)


@pytest.mark.parametrize("G", [1, 2])
def test_rsim_tma_ring_cycles(cel, G):
    """rsim_row_tma's 4-stage mbarrier ring (16 rows per stage) refills and
    flips phase once t > 48: T = 140 rows runs ceil(139/16) = 9 stages per
    launch at the end, > 2 full ring cycles, at W = 1000 >= 2 * 148 (the TMA
    kernel's precondition), bit-exact against the oracle."""
    run_both(cel, P.rsim(1000, 140), G, "auto")


def test_rsim_register_kernel(cel, monkeypatch):
    """The register fallback rsim_row_kernel<16> (CEL_RSIM=0 selects it for the
    runtime; otherwise taken when the TMA preconditions fail): rows t >= 16
    run its unrolled 16-load loop plus the tail, bit-exact."""
    monkeypatch.setenv("CEL_RSIM", "0")
    run_both(cel, P.rsim(1000, 40), 2, "auto")
    run_both(cel, P.rsim(301, 37), 1, "none")


def test_jacobi_lsu_kernel(cel, monkeypatch):
    """The LSU fallback jacobi7_vec (CEL_JACOBI=l; otherwise taken when the
    allocation is not TMA-compatible), bit-exact."""
    monkeypatch.setenv("CEL_JACOBI", "l")
    run_both(cel, P.jacobi3d(36, 4), 4)
    run_both(cel, P.jacobi3d(20, 3), 1)


@pytest.mark.parametrize("G", [2, 4])
@pytest.mark.parametrize("dma", [True, False])
def test_forced_peer_path(cel, G, dma, monkeypatch):
    """CEL_FORCE_PEER=1: copies between virtual devices of one GPU take the
    path of copies between GPUs -- with dma, the copy-engine plan (1-D runs
    and pitched 2-D boxes <= 4 MiB: cudaMemcpyAsync / cudaMemcpy2DAsync pitch
    arithmetic), without (CEL_PEER_DMA=0, what pushes > 4 MiB take) the fenced
    persistent-grid peer copy kernel -- so one B200 covers that code: 3-D halo
    faces, ragged and 2-D-split WaveSim, N-body / RSim gathers and random
    programs, bit-exact and with the oracle's instruction log."""
    monkeypatch.setenv("CEL_FORCE_PEER", "1")
    monkeypatch.setenv("CEL_COLL_P2P", "0")          # gathers too: as the pushes they are
    if not dma:
        monkeypatch.setenv("CEL_PEER_DMA", "0")
    run_both(cel, P.jacobi3d(36, 4), G)
    run_both(cel, P.jacobi3d(20, 3), G + 1)
    run_both(cel, P.wavesim(1040, 7, rows=300), G)
    run_both(cel, P.wavesim(515, 5, rows=130, split="2d", mapper="neighborhood_axes"), G)
    st = run_both(cel, P.nbody(1000, 2), G).final_stats
    assert st["copies_coherence"] > 0 and (st["copy_launches"] == 0) == dma
    run_both(cel, P.rsim(1000, 24), G, "none")
    for s in range(6):
        run_both(cel, P.random_program(7100 + 11 * G + s), G, arena=32 << 20)


@pytest.mark.parametrize("G", [2, 4])
def test_tma_tensor_map_copies(cel, G, monkeypatch):
    """CEL_COPY=tma: strided boxes of copies within a GPU whose rows start and
    end on 16-byte boundaries (3-D y-faces, resize copies of rows at a pitch)
    move by TMA tensor maps (UTMALDG / UTMASTG, tiles clipped at the box edge
    by maps cut there); the rest of each program stays on the LSU kernel;
    bit-exact with the oracle's bytes and log."""
    monkeypatch.setenv("CEL_COPY", "tma")
    monkeypatch.setenv("CEL_NO_GROW", "1")
    st = run_both(cel, P.jacobi3d(36, 4), G).final_stats
    assert (st["tma_copy_launches"] > 0) == (G == 4)          # 2 x 1 tiles have contiguous z-faces only
    run_both(cel, P.jacobi3d(20, 3), G + 1)
    # 2-D tiles: row halos are one run, column halos one element wide (TMA
    # needs 16-byte aligned row segments): these stay on the LSU kernel
    run_both(cel, P.wavesim(515, 5, rows=130, split="2d", mapper="neighborhood_axes"), G)
    run_both(cel, P.wavesim(516, 4, rows=260, split="2d"), G, "none")
    for s in range(6):
        run_both(cel, P.random_program(7300 + 11 * G + s), G, "none", arena=32 << 20)


@pytest.mark.parametrize("fuse", [True, False])
def test_rsim_rows_fused_with_gathers(cel, fuse, monkeypatch):
    """An RSim row's all-gather (the next task's coherence copy set) fused into
    the row kernel that produces it: the executor holds the row kernel until
    the set arrives and launches it with a peer epilogue (stores into every
    receiver's allocation, then gather counters); otherwise (CEL_FUSE_ROWS=0)
    the set runs as P2P gather kernels.  Bit-exact with the oracle's bytes
    and log, on virtual devices of one GPU (and on distinct GPUs when there)."""
    if not fuse:
        monkeypatch.setenv("CEL_FUSE_ROWS", "0")
    for G in (2, 4):
        st = run_both(cel, P.rsim(1000, 40), G).final_stats
        assert st["gather_sets"] > 0 and st["coll_p2p"] + st["coll_fused"] == st["gather_sets"]
        assert (st["coll_fused"] > st["gather_sets"] // 2) == fuse, (st["coll_fused"], st["gather_sets"])
    run_both(cel, P.rsim(1000, 140), 3)                      # ring cycles of the TMA kernel, fused
    run_both(cel, P.rsim(1000, 24), 2, "none")               # growing allocations
    n = torch.cuda.device_count()
    if n >= 2:
        run_both(cel, P.rsim(84000, 48), n, devices=list(range(n)))


def test_all_gather_collective_vs_pushes(cel, monkeypatch):
    """§8 a7: the same programs with the all-gather copy sets run as NCCL
    broadcasts and as peer pushes give identical bytes."""
    monkeypatch.setenv("CEL_COLL_MIN_BYTES", "0")
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    devs = list(range(n))
    for prog in (P.nbody(3000, 3), P.rsim(3001, 12), P.nbody(777, 2, host_init=True)):
        for coll in (True, False):
            rt = cel.Runtime(n, cuda_devices=devs, arena_bytes=256 << 20, collective=coll)
            rt.profile_enable(True)         # profile events on every device (collective groups included)
            got = [r[1] for r in run_program(rt, prog) if r[0] == "read"]
            o = OracleRuntime(n)
            run_program(o, prog)
            exp = simulate(o)
            for k, arr in enumerate(got):
                defined = exp[k] != np.uint32(0x7FC00BAD)
                assert np.array_equal(arr[defined], exp[k][defined]), (prog["name"], coll, k)


def test_all_gather_multicast(cel, monkeypatch):
    """with CEL_COLL_MC=1 (one process, distinct GPUs, VMM
    allocations) every all-gather set runs as multicast stores through one
    NVLS object bound to the G receiving allocations, completed by a
    multicast flag: RSim rows (84 KB-class sets) bit-exact against the oracle,
    and N-body at 2^17 bodies (2 MiB of positions per device) bit-identical to
    the single-GPU run of the same program (the oracle-sampled path)."""
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    monkeypatch.setenv("CEL_COLL_MC", "1")
    monkeypatch.setenv("CEL_FUSE_ROWS", "0")           # (fused rows would take RSim's sets first)
    devs = list(range(n))
    st = run_both(cel, P.rsim(8000, 80), n, devices=devs).final_stats
    assert st["coll_multicast"] == st["gather_sets"] > 0
    st = run_both(cel, P.rsim(40000, 24), n, "none", devices=devs).final_stats   # growing VMM allocations: rebinding
    assert st["coll_multicast"] > 0
    N = 1 << 17
    prog = P.nbody(N, 2)
    rt = cel.Runtime(n, cuda_devices=devs, arena_bytes=256 << 20)
    got = [r[1] for r in run_program(rt, prog) if r[0] == "read"]
    monkeypatch.setenv("CEL_COLL_MC", "0")
    rt1 = cel.Runtime(1, arena_bytes=256 << 20)
    ref = [r[1] for r in run_program(rt1, prog) if r[0] == "read"]
    for a, b in zip(got, ref):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("grow", [True, False])
def test_rsim_in_place_growth(cel, grow, monkeypatch):
    """Without lookahead every RSim row resizes the allocation (alloc -> copy ->
    free).  In-place growth takes the old allocation's address, so the
    resize copies move nothing; results and the instruction log are unchanged."""
    if not grow:
        monkeypatch.setenv("CEL_NO_GROW", "1")
    for G in (1, 2):
        st = run_both(cel, P.rsim(1000, 24), G, "none").final_stats
        assert st["copies_resize"] > 0
        assert (st["copies_elided"] > 0) == grow
        assert st["copies_elided"] <= st["copies_resize"]


@pytest.mark.parametrize("vmm", [True, False])
def test_vmm_growth_interleaved(cel, vmm, monkeypatch):
    """SURVEY NEXT-3 / P:L549-556: two buffers growing in turn without
    lookahead.  The arena can only grow an allocation in place when the range
    right after it is free, which the other buffer's allocation blocks: every
    resize copies.  With VMM (single process) a resize that cannot grow in
    the arena gets an allocation with its own address range reserved up to
    the buffer's end, so after one real copy per buffer every later resize
    maps granules behind the rows and its copy is elided.  Same instruction
    log and bytes either way."""
    if not vmm:
        monkeypatch.setenv("CEL_NO_VMM", "1")
    st = run_both(cel, P.rsim_pair(600000, 10), 1, "none", arena=512 << 20).final_stats
    info = (st["copies_resize"], st["copies_elided"], st["vmm_maps"])
    assert st["copies_resize"] > 0, info
    # (a resize copies one fragment per original producer of the old rows, R9)
    if vmm:
        assert st["copies_elided"] >= 0.8 * st["copies_resize"] and st["vmm_maps"] > 2, info
    else:
        assert st["copies_elided"] < 0.8 * st["copies_resize"] and st["vmm_maps"] == 0, info
    st = run_both(cel, P.rsim(600000, 12), 2, "none", arena=512 << 20).final_stats
    info = (st["copies_resize"], st["copies_elided"], st["vmm_maps"])
    assert st["copies_elided"] >= 0.8 * st["copies_resize"], info


def test_arena_overflow_maps_vmm(cel):
    """The arena size caps nothing in one process: allocations that do not fit
    the arena are VMM-mapped (here a 64 MiB arena and two 128 MiB fields)."""
    st = run_both(cel, P.wavesim(8192, 3, rows=4096), 2, arena=64 << 20).final_stats
    assert st["vmm_maps"] > 0


def test_physical_multi_gpu(cel, monkeypatch):
    monkeypatch.setenv("CEL_COLL_MIN_BYTES", "0")     # small test gathers take the NCCL path too
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    devs = list(range(n))
    run_both(cel, P.wavesim(1024, 7, rows=600), n, devices=devs)
    st = run_both(cel, P.nbody(2048, 2), n, devices=devs).final_stats
    # the `all` gather of P runs as grouped NCCL broadcasts (§8 a7)
    assert st["gather_sets"] == 2 and st["coll_groups"] == 2 and st["coll_copies"] == st["copies_coherence"]
    run_both(cel, P.jacobi3d(40, 3), n, devices=devs)
    st = run_both(cel, P.rsim(2000, 16), n, "none", devices=devs).final_stats
    assert st["coll_groups"] == st["gather_sets"] > 0
    for s in range(6):
        run_both(cel, P.random_program(500 + s), n, devices=devs, arena=32 << 20)


# ---------------------------------------------------------------- full size
def light_cone_wave(rows_lo, rows_hi, n, steps, seed=2):
    """Oracle values of rows [rows_lo, rows_hi) of the 16384^2 WaveSim after
    `steps` steps, computed on the light cone only (rows +- steps)."""
    a = max(0, rows_lo - steps - 1)
    b = min(n, rows_hi + steps + 1)
    ext = g.box([0, 0], [n, n])
    box = g.box([a, 0], [b, n])
    i0 = np.arange(a, b, dtype=np.uint64)[:, None] * np.uint64(n) + np.arange(n, dtype=np.uint64)[None, :]
    f = init_value(seed, i0).reshape(b - a, n, 1, 1)
    u = Acc(f.view(np.uint32).copy(), box, ext)
    up = Acc(f.view(np.uint32).copy(), box, ext)
    lo, hi = a, b
    for k in range(steps):
        lo2 = lo if lo == 0 else lo + 1
        hi2 = hi if hi == n else hi - 1
        wb = g.box([lo2, 0], [hi2, n])
        if k % 2 == 0:
            k_wave5({}, [wb, wb], [u, up])
        else:
            k_wave5({}, [wb, wb], [up, u])
        lo, hi = lo2, hi2
    last = up if steps % 2 == 1 else u
    return last.arr[rows_lo - a:rows_hi - a]


@pytest.mark.parametrize("G", [1, 2])
def test_wavesim_full_size_sampled(cel, G):
    """BASELINE config 2 at full size (16384^2), the bench's launch
    configuration: sampled rows at the global edges and device boundaries."""
    n, steps = 16384, 5
    rt = cel.Runtime(G, cuda_devices=[0] * G, arena_bytes=int(2 * (n // G + 2) * n * 4 * 1.05) + (256 << 20))
    u = rt.buffer_create(2, [n, n], 4)
    up = rt.buffer_create(2, [n, n], 4)
    for op in P.wavesim_init(n):
        rt.task_submit(op[1])
    for k in range(steps):
        rt.task_submit(P.wavesim_step(n, k)[1])
    last = up if steps % 2 == 1 else u
    samples = [(0, 8), (n // 2 - 4, n // 2 + 4), (n - 8, n), (5000, 5003)]
    for lo, hi in samples:
        got = rt.buffer_read(last, ([lo, 0], [hi, n]))
        exp = light_cone_wave(lo, hi, n, steps)
        assert np.array_equal(got, exp), (lo, hi)
    rt.shutdown()


def test_nbody_full_size_sampled(cel):
    """BASELINE config 3 at 2^20 bodies: one timestep, 16 sampled bodies
    bit-exact (sequential sum over 2^20 bodies in the oracle)."""
    N = 1 << 20
    rt = cel.Runtime(1, arena_bytes=256 << 20)
    prog = P.nbody(N, steps=0)
    Pb = rt.buffer_create(1, [N], 16)
    Vb = rt.buffer_create(1, [N], 16)
    for op in prog["ops"]:
        if op[0] == "task":
            rt.task_submit(op[1])
    rt.task_submit(P.nbody(N, 1)["ops"][2][1])          # the timestep task
    v = rt.buffer_read(Vb, ([0], [N])).view(np.float32)[:, 0, 0, :]
    pos = init_value(3, np.arange(4 * N, dtype=np.uint64)).reshape(N, 4)[:, :3].astype(np.float32)
    c = np.float32(2.0 ** -7) * np.float32(2.0 ** -20)
    rng = np.random.default_rng(0)
    for i in list(rng.integers(0, N, 14)) + [0, N - 1]:
        a = nbody_accel_one(pos, pos[i])
        assert np.array_equal(v[i, :3], np.float32(0) + c * a), i
    rt.shutdown()


def test_nbody_fast_math_within_tolerance(cel):
    """fast_math (FMA + rsqrt) N-body: not bit-exact by design (R16).  The
    bar is R16's performance-build tolerance, north_star's "1e-6 relative"
    read as |g - o| <= 1e-6 * max(|o|, max |field|) per component, against
    the oracle's exact sequential float32 result."""
    N = 4096
    prog = P.nbody(N, 1)
    rt = cel.Runtime(2, cuda_devices=[0, 0], arena_bytes=64 << 20, fast_math=True)
    got = [r[1] for r in run_program(rt, prog) if r[0] == "read"]
    o = OracleRuntime(2)
    run_program(o, prog)
    exp = simulate(o)
    for k in (0, 1):                                          # P and V after the step
        vg = got[k].view(np.float32)[:, 0, 0, :3].astype(np.float64)
        vo = exp[k].view(np.float32)[:, 0, 0, :3].astype(np.float64)
        scale = np.maximum(np.abs(vo), np.abs(vo).max())
        err = (np.abs(vg - vo) / scale).max()
        print("fast_math readback %d: max |g-o| / max(|o|, max|field|) = %.3g" % (k, err))
        assert err <= 1e-6, err
    assert not np.array_equal(got[1], exp[1]), "fast_math path did not run (bit-identical to the exact kernel)"


def light_cone_jacobi(z_lo, z_hi, n, steps, seed=5):
    """Oracle planes [z_lo, z_hi) of the 1024^3 Jacobi after `steps` steps,
    computed on the light cone only (planes +- steps, full y/x)."""
    from oracle.kernels import k_jacobi7
    a = max(0, z_lo - steps - 1)
    b = min(n, z_hi + steps + 1)
    ext = g.box([0, 0, 0], [n, n, n])
    box = g.box([a, 0, 0], [b, n, n])
    z = np.arange(a, b, dtype=np.uint64)[:, None, None]
    y = np.arange(n, dtype=np.uint64)[None, :, None]
    x = np.arange(n, dtype=np.uint64)[None, None, :]
    f = init_value(seed, (z * np.uint64(n) + y) * np.uint64(n) + x).reshape(b - a, n, n, 1)
    A = Acc(f.view(np.uint32).copy(), box, ext)
    B = Acc(np.zeros_like(A.arr), box, ext)
    lo, hi = a, b
    for k in range(steps):
        lo2 = lo if lo == 0 else lo + 1
        hi2 = hi if hi == n else hi - 1
        wb = g.box([lo2, 0, 0], [hi2, n, n])
        if k % 2 == 0:
            k_jacobi7({}, [wb, wb], [A, B])
        else:
            k_jacobi7({}, [wb, wb], [B, A])
        lo, hi = lo2, hi2
    last = B if steps % 2 == 1 else A
    return last.arr[z_lo - a:z_hi - a]


@pytest.mark.parametrize("G", [1, 4])
def test_jacobi_full_size_sampled(cel, G):
    """BASELINE config 5 at full size (1024^3, TMA kernel, 2-D split over G
    virtual devices): sampled planes at the global edges, the split boundary
    and the interior, bit-exact."""
    n, steps = 1024, 3
    rt = cel.Runtime(G, cuda_devices=[0] * G, arena_bytes=int(2 * n ** 3 * 4 / G * 1.25) + (512 << 20))
    prog = P.jacobi3d(n, steps)
    rt.buffer_create(3, [n, n, n], 4)
    rt.buffer_create(3, [n, n, n], 4)
    for op in prog["ops"]:
        if op[0] == "task":
            rt.task_submit(op[1])
    last = 1 if steps % 2 == 1 else 0
    for lo, hi in [(0, 2), (n // 2 - 1, n // 2 + 1), (n - 2, n), (333, 334)]:
        got = rt.buffer_read(last, ([lo, 0, 0], [hi, n, n]))
        exp = light_cone_jacobi(lo, hi, n, steps)
        assert np.array_equal(got, exp), (lo, hi)
    rt.shutdown()


def test_rsim_full_width(cel):
    """BASELINE config 4 at its full width W = 84,000 (T = 48 rows, 4 devices,
    lookahead none and auto): the whole buffer bit-exact against the oracle."""
    prog = P.rsim(84000, 48)
    for mode in ("none", "auto"):
        run_both(cel, prog, 4, mode, arena=256 << 20)


# ------------------------------------------------------------ §4.4 accessor bounds checking
def test_bounds_check_reports_out_of_range_accesses(cel):
    """a 3-point stencil declared with a one_to_one read (instead of
    neighborhood(1)) reads one element past each chunk: the runtime reports the
    bounding box of the offending accesses after the kernel exits."""
    n = 4096
    prog = {"name": "oob", "buffers": [{"dims": 1, "extent": [n], "elem_size": 4, "host_init": None},
                                       {"dims": 1, "extent": [n], "elem_size": 4, "host_init": None}],
            "ops": [P._task(1, P.full([n]), "fill_hash", [(0, "write", ("one_to_one",))], {"seed": 7}),
                    P._task(1, P.full([n]), "stencil3", [(0, "read", ("one_to_one",)),
                                                         (1, "write", ("one_to_one",))])]}
    rt = cel.Runtime(2, cuda_devices=[0, 0], arena_bytes=64 << 20, bounds_check=True)
    for b in prog["buffers"]:
        rt.buffer_create(b["dims"], b["extent"], b["elem_size"])
    with pytest.raises(cel.CelError) as e:
        for op in prog["ops"]:
            rt.task_submit(op[1])
        rt.wait()
    assert e.value.code == -2
    msg = str(e.value)
    # device 0 owns [0, 2048): its only out-of-range read is element 2048
    assert "accessor out of bounds" in msg and "device 0, accessor 0" in msg
    assert "[[2048,0,0],[2049,1,1]]" in msg and "[[0,0,0],[2048,1,1]]" in msg
    with pytest.raises(cel.CelError):       # sticky: the runtime is poisoned
        rt.wait()


@pytest.mark.parametrize("G", [1, 2, 3])
def test_bounds_check_no_false_positives(cel, G):
    """Zero false positives on the paper's workloads and random probe
    programs; with checking on the kernels take their scalar paths, so this is
    also parity of those paths."""
    progs = [P.c1_chain(4096), P.wavesim(515, 5, rows=130), P.jacobi3d(24, 3), P.nbody(700, 2), P.rsim(1000, 12),
             P.nbody(300, 2, host_init=True)] + [P.random_program(8800 + 5 * G + s) for s in range(6)]
    for prog in progs:
        rt = cel.Runtime(G, cuda_devices=[0] * G, arena_bytes=64 << 20, bounds_check=True)
        got = [r[1] for r in run_program(rt, prog) if r[0] == "read"]
        o = OracleRuntime(G)
        run_program(o, prog)
        exp = simulate(o)
        for k, arr in enumerate(got):
            defined = exp[k] != np.uint32(0x7FC00BAD)
            assert np.array_equal(arr[defined], exp[k][defined]), prog["name"]


@pytest.mark.parametrize("G", [2, 4])
def test_wavesim_2d_split_axis_neighborhood(cel, G):
    """WaveSim with the 2-D split, box and axis-only
    neighbourhoods, bit-exact against the oracle (ragged tiles)."""
    for mp in ("neighborhood", "neighborhood_axes"):
        run_both(cel, P.wavesim(515, 5, rows=130, split="2d", mapper=mp), G)
        run_both(cel, P.wavesim(516, 4, rows=260, split="2d", mapper=mp), G)


@pytest.mark.parametrize("mode", ["none", "auto"])
def test_degenerate_shapes(cel, mode):
    """Empty device chunks (fewer rows / bodies than devices), 1x1 grids,
    one-element buffers and a 2x4 grid under the 2-D split: bit-exact, and the
    same instruction log as the oracle."""
    cases = [(P.wavesim(5, 3, rows=3), 4), (P.wavesim(1, 3, rows=1), 2), (P.nbody(1, 2), 2), (P.nbody(3, 2), 4),
             (P.jacobi3d(2, 2), 3), (P.rsim(3, 4), 4), (P.c1_chain(2), 4),
             (P.wavesim(4, 2, rows=2, split="2d", mapper="neighborhood_axes"), 4)]
    for prog, G in cases:
        run_both(cel, prog, G, mode, arena=8 << 20)
