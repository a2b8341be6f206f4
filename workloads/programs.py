"""Program descriptions for the five BASELINE.json configs and random tests.

A program is plain data, fed by `workloads.driver.run_program` to the oracle
and to the product binding alike:

  {"buffers": [{"dims", "extent", "elem_size", "host_init": ndarray | None}],
   "ops": [("task", spec) | ("wait",) | ("read", bid, (mins, maxs)) |
           ("destroy", bid)]}
  spec = {"dims", "range": (mins, maxs), "split": "1d" | "2d",
          "kernel": name, "params": {...},
          "accesses": [(bid, "read" | "write" | "read_write", mapper)]}
  mapper = ("one_to_one",) | ("neighborhood", (b0, b1, b2)) | ("neighborhood_axes", (b0, b1, b2)) | ("all",) |
           ("fixed", (mins, maxs)) | ("remap", (mins, maxs), (k0, k1, k2))

Input recipe: every value is either produced on the
device by the counter-based `fill_hash` kernel (seed = config index + 1) or,
for host-initialised buffers, drawn here from numpy's PCG64 with a fixed seed.
"""

import numpy as np


def init_values(seed, idx):
    """The synthetic input recipe's value of element word `idx` (uint64 array):
    init(seed, i) = 2 * (float)(splitmix64(seed + i) >> 40) * 2^-24 - 1, exact
    in [-1, 1).  The device fill_hash kernel and the oracle
    implement it independently; this copy lets harnesses byte-check data that
    a copy moved without running either side."""
    M = np.uint64(0xFFFFFFFFFFFFFFFF)
    with np.errstate(over="ignore"):
        z = (np.asarray(idx, dtype=np.uint64) + np.uint64(seed) + np.uint64(0x9E3779B97F4A7C15)) & M
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    v = (z >> np.uint64(40)).astype(np.float32)
    return (np.float32(2.0) * (v * np.float32(2.0 ** -24))) - np.float32(1.0)


def _task(dims, rng, kernel, accesses, params=None, split="1d"):
    return ("task", {"dims": dims, "range": rng, "split": split, "kernel": kernel,
                     "params": dict(params or {}), "accesses": list(accesses)})


def full(extent):
    return ([0] * len(extent), list(extent))


# ---------------------------------------------------------------- C1
def c1_chain(n=4096, seed=1):
    """Config 1: 1-D buffer of n floats, 4-task chain (one_to_one write,
    neighborhood(1) read) — the Listing 5 pattern."""
    A, B = 0, 1
    r = full([n])
    ops = [
        _task(1, r, "fill_hash", [(A, "write", ("one_to_one",))], {"seed": seed}),
        _task(1, r, "stencil3", [(A, "read", ("neighborhood", (1,))), (B, "write", ("one_to_one",))]),
        _task(1, r, "stencil3", [(B, "read", ("neighborhood", (1,))), (A, "write", ("one_to_one",))]),
        _task(1, r, "stencil3", [(A, "read", ("neighborhood", (1,))), (B, "write", ("one_to_one",))]),
        ("read", B, r),
        ("destroy", A),
        ("destroy", B),
    ]
    bufs = [{"dims": 1, "extent": [n], "elem_size": 4, "host_init": None} for _ in range(2)]
    return {"name": "c1_chain", "buffers": bufs, "ops": ops}


def listing5(n=64, seed=1):
    """Listing 5: one_to_one write, then a read of the one-neighborhood."""
    A, B = 0, 1
    r = full([n])
    ops = [
        _task(1, r, "fill_hash", [(A, "write", ("one_to_one",))], {"seed": seed}),
        _task(1, r, "stencil3", [(A, "read", ("neighborhood", (1,))), (B, "write", ("one_to_one",))]),
        ("read", B, r),
    ]
    bufs = [{"dims": 1, "extent": [n], "elem_size": 4, "host_init": None} for _ in range(2)]
    return {"name": "listing5", "buffers": bufs, "ops": ops}


# ---------------------------------------------------------------- C2
def wavesim_init(n, seed=2, rows=None, split="1d"):
    rows = n if rows is None else rows
    u, up = 0, 1
    r = full([rows, n])
    return [
        _task(2, r, "fill_hash", [(u, "write", ("one_to_one",))], {"seed": seed}, split=split),
        _task(2, r, "fill_hash", [(up, "write", ("one_to_one",))], {"seed": seed}, split=split),
    ]


def wavesim_step(n, k, rows=None, split="1d", mapper="neighborhood"):
    """Step k of WaveSim: up = wave5(u, up); then the roles swap.
    mapper "neighborhood_axes" declares the 5-point stencil's cross exactly
    (no corners); split "2d" tiles the grid over the devices."""
    rows = n if rows is None else rows
    u, up = (0, 1) if k % 2 == 0 else (1, 0)
    return _task(2, full([rows, n]), "wave5",
                 [(u, "read", (mapper, (1, 1))), (up, "read_write", ("one_to_one",))], split=split)


def wavesim(n=16384, steps=4, seed=2, rows=None, split="1d", mapper="neighborhood"):
    """Config 2: WaveSim 2-D 5-point stencil, rows x n fp32, 1-D row split
    (split / mapper: the NEXT-3 variants, see wavesim_step)."""
    rows = n if rows is None else rows
    ops = wavesim_init(n, seed, rows, split) + [wavesim_step(n, k, rows, split, mapper) for k in range(steps)]
    ops += [("read", 0, full([rows, n])), ("read", 1, full([rows, n]))]
    bufs = [{"dims": 2, "extent": [rows, n], "elem_size": 4, "host_init": None} for _ in range(2)]
    return {"name": "wavesim", "buffers": bufs, "ops": ops}


# ---------------------------------------------------------------- C3
def nbody(n=1 << 20, steps=2, seed=3, host_init=False):
    """Config 3 / Listing 1: timestep (P read all, V read_write
    one_to_one) + update (V read, P read_write) per step; float4 bodies."""
    P, V = 0, 1
    r = full([n])
    ops = []
    bufs = [{"dims": 1, "extent": [n], "elem_size": 16, "host_init": None} for _ in range(2)]
    if host_init:
        g = np.random.default_rng(seed)
        p = g.uniform(-1.0, 1.0, size=(n, 4)).astype(np.float32)
        p[:, 3] = 0.0
        bufs[0]["host_init"] = p
        bufs[1]["host_init"] = np.zeros((n, 4), dtype=np.float32)
    else:
        ops.append(_task(1, r, "fill_hash", [(P, "write", ("one_to_one",))], {"seed": seed}))
        ops.append(_task(1, r, "fill_const", [(V, "write", ("one_to_one",))], {"value": 0.0}))
    for _ in range(steps):
        ops.append(_task(1, r, "nbody_step", [(P, "read", ("all",)), (V, "read_write", ("one_to_one",))]))
        ops.append(_task(1, r, "nbody_update", [(V, "read", ("one_to_one",)), (P, "read_write", ("one_to_one",))]))
    ops += [("read", P, r), ("read", V, r)]
    return {"name": "nbody", "buffers": bufs, "ops": ops}


# ---------------------------------------------------------------- C4
def rsim_row(W, t):
    return _task(1, full([W]), "rsim_row",
                 [(0, "read", ("fixed", ([0, 0], [t, W]))),
                  (0, "write", ("remap", ([t, 0], [t + 1, 0]), (-1, 0, -1)))], {"t": t})


def rsim(W=84000, T=1024, seed=4):
    """Config 4: RSim-shaped growth: row t reads rows [0,t) and
    appends row t; the kernel index space is the W columns."""
    ops = [_task(1, full([W]), "fill_hash", [(0, "write", ("remap", ([0, 0], [1, 0]), (-1, 0, -1)))],
                 {"seed": seed})]
    ops += [rsim_row(W, t) for t in range(1, T)]
    ops.append(("read", 0, full([T, W])))
    bufs = [{"dims": 2, "extent": [T, W], "elem_size": 4, "host_init": None}]
    return {"name": "rsim", "buffers": bufs, "ops": ops}


def rsim_pair(W, T, seed=4):
    """Two RSim-shaped buffers growing in turn (row t of A, then row t of B):
    without lookahead every task resizes its buffer's allocation while the
    other buffer's allocation sits right behind it."""
    ops = []
    for b in (0, 1):
        ops.append(_task(1, full([W]), "fill_hash", [(b, "write", ("remap", ([0, 0], [1, 0]), (-1, 0, -1)))],
                         {"seed": seed + b}))
    for t in range(1, T):
        for b in (0, 1):
            ops.append(_task(1, full([W]), "rsim_row",
                             [(b, "read", ("fixed", ([0, 0], [t, W]))),
                              (b, "write", ("remap", ([t, 0], [t + 1, 0]), (-1, 0, -1)))], {"t": t}))
    ops += [("read", 0, full([T, W])), ("read", 1, full([T, W]))]
    bufs = [{"dims": 2, "extent": [T, W], "elem_size": 4, "host_init": None} for _ in range(2)]
    return {"name": "rsim_pair", "buffers": bufs, "ops": ops}


# ---------------------------------------------------------------- C5
def jacobi_step(n, k):
    a, b = (0, 1) if k % 2 == 0 else (1, 0)
    return _task(3, full([n, n, n]), "jacobi7",
                 [(a, "read", ("neighborhood", (1, 1, 1))), (b, "write", ("one_to_one",))], split="2d")


def jacobi3d(n=1024, steps=2, seed=5):
    """Config 5: 3-D 7-point stencil n^3 fp32, 2-D split (z, y)."""
    ops = [_task(3, full([n, n, n]), "fill_hash", [(0, "write", ("one_to_one",))], {"seed": seed}, split="2d")]
    ops += [jacobi_step(n, k) for k in range(steps)]
    last = steps % 2 == 1
    ops.append(("read", 1 if last else 0, full([n, n, n])))
    bufs = [{"dims": 3, "extent": [n, n, n], "elem_size": 4, "host_init": None} for _ in range(2)]
    return {"name": "jacobi3d", "buffers": bufs, "ops": ops}


# ---------------------------------------------------------------- random
def random_program(seed, max_tasks=10):
    """Random small program of u32 `probe` tasks over 1-3 same-shaped buffers.
    A task writes one buffer (one_to_one, write or read_write) and reads up to
    two OTHER buffers with random mappers; waits / readbacks interleave."""
    g = np.random.default_rng(seed)
    dims = int(g.integers(1, 4))
    ext = [int(g.integers(3, {1: 40, 2: 12, 3: 7}[dims])) for _ in range(dims)]
    nb = int(g.integers(1, 4))
    bufs = []
    ops = []
    for b in range(nb):
        hi = None
        if g.random() < 0.5:
            hi = g.integers(0, 2 ** 32, size=ext, dtype=np.uint32)
        bufs.append({"dims": dims, "extent": list(ext), "elem_size": 4, "host_init": hi})
    for b in range(nb):
        if bufs[b]["host_init"] is None:
            ops.append(_task(dims, full(ext), "probe", [(b, "write", ("one_to_one",))],
                             {"salt": int(g.integers(0, 2 ** 31))}, split="1d"))

    def rbox():
        mn, mx = [], []
        for e in ext:
            a = int(g.integers(0, e))
            c = int(g.integers(a + 1, e + 1))
            mn.append(a)
            mx.append(c)
        return (mn, mx)

    for _ in range(int(g.integers(2, max_tasks + 1))):
        r = g.random()
        if r < 0.08:
            ops.append(("wait",))
            continue
        if r < 0.18:
            ops.append(("read", int(g.integers(0, nb)), rbox()))
            continue
        w = int(g.integers(0, nb))
        rng = full(ext) if g.random() < 0.7 else rbox()
        acc = [(w, "read_write" if g.random() < 0.4 else "write", ("one_to_one",))]
        others = [b for b in range(nb) if b != w]
        g.shuffle(others)
        for b in others[:int(g.integers(0, 3))]:
            k = g.random()
            if k < 0.3:
                mp = ("one_to_one",)
            elif k < 0.65:
                mp = ("neighborhood", tuple(int(g.integers(0, 3)) for _ in range(dims)))
            elif k < 0.85:
                mp = ("all",)
            else:
                mp = ("fixed", rbox())
            acc.append((b, "read", mp))
        g.shuffle(acc)
        split = "2d" if dims >= 2 and g.random() < 0.4 else "1d"
        ops.append(_task(dims, rng, "probe", acc, {"salt": int(g.integers(0, 2 ** 31))}, split=split))
    for b in range(nb):
        ops.append(("read", b, full(ext)))
    return {"name": "random%d" % seed, "buffers": bufs, "ops": ops}
