"""Synthetic workload arithmetic in NumPy (test infrastructure; oracle).

The paper's listings are missing (Listing 1, Listing 5) and
WaveSim's formula is not given, so the kernels are DESIGN.md
readings with dyadic constants (SURVEY §8(c) "Synthetic workloads").  R16:
fp32, IEEE round-to-nearest-even, every operation written out in the order
the CUDA kernels use; NumPy float32 elementwise ops are single IEEE ops (no
FMA, no reassociation), sequential sums are explicit loops / cumsum.

Data model: every allocation is a 4-D uint32 array (n0, n1, n2, words) over
its box, words = elem_size/4; kernels view it as float32 where the workload
is floating point.  An accessor is (array, alloc_box); kernels address it by
global buffer coordinates, so the same function serves the per-device
simulation (allocation arrays) and the sequential definition (one global
array per buffer).
"""

import numpy as np

from . import geometry as g

F32 = np.float32
U32 = np.uint32
U64 = np.uint64


# ------------------------------------------------------------ generators
def splitmix64(x):
    """Vigna's SplitMix64 output function applied to state x (uint64 array):
    z = x + 0x9E3779B97F4A7C15; z ^= z>>30; z *= 0xBF58476D1CE4E5B9;
    z ^= z>>27; z *= 0x94D049BB133111EB; z ^= z>>31."""
    with np.errstate(over="ignore"):
        z = np.asarray(x, dtype=U64) + U64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> U64(30))) * U64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> U64(27))) * U64(0x94D049BB133111EB)
        return z ^ (z >> U64(31))


def init_value(seed, idx):
    """init(seed, i) = 2*(float)(splitmix64(seed+i) >> 40)*2^-24 - 1, exact in [-1,1)."""
    with np.errstate(over="ignore"):
        h = splitmix64(U64(seed) + np.asarray(idx, dtype=U64))
    v = (h >> U64(40)).astype(F32)
    return (F32(2.0) * (v * F32(2.0 ** -24))) - F32(1.0)


def fmix32(h):
    """MurmurHash3 32-bit finaliser on uint32 arrays."""
    with np.errstate(over="ignore"):
        h = np.asarray(h, dtype=U32)
        h = h ^ (h >> U32(16))
        h = h * U32(0x85EBCA6B)
        h = h ^ (h >> U32(13))
        h = h * U32(0xC2B2AE35)
        return h ^ (h >> U32(16))


# ------------------------------------------------------------ accessors
class Acc:
    """Accessor over an allocation ("allocation pointers are
    interpolated into accessors")."""

    def __init__(self, arr, box, extent):
        self.arr = arr
        self.box = box
        self.extent = extent

    def gather(self, i0, i1, i2):
        b = self.box[0]
        return self.arr[np.ix_(np.asarray(i0) - b[0], np.asarray(i1) - b[1], np.asarray(i2) - b[2])]

    def view_box(self, bx):
        b = self.box[0]
        return self.arr[bx[0][0] - b[0]:bx[1][0] - b[0],
                        bx[0][1] - b[1]:bx[1][1] - b[1],
                        bx[0][2] - b[2]:bx[1][2] - b[2]]

    def f32(self, i0, i1, i2):
        return self.gather(i0, i1, i2).view(F32)

    def store(self, bx, words):
        self.view_box(bx)[...] = words


def _ar(bx, d):
    return np.arange(bx[0][d], bx[1][d], dtype=np.int64)


def _clip(a, n):
    return np.clip(a, 0, n - 1)


# ------------------------------------------------------------ kernels
def k_fill_hash(p, boxes, accs):
    """FILL_HASH: word w of element x gets init(seed, lin(x)*words + w)."""
    bx, a = boxes[0], accs[0]
    if g.is_empty(bx):
        return
    E = g.shape(a.extent)
    words = a.arr.shape[3]
    i0, i1, i2 = np.meshgrid(_ar(bx, 0), _ar(bx, 1), _ar(bx, 2), indexing="ij")
    lin = ((i0 * E[1]) + i1) * E[2] + i2
    idx = lin[..., None] * words + np.arange(words)
    a.store(bx, init_value(p["seed"], idx.astype(np.uint64)).view(U32))


def k_fill_const(p, boxes, accs):
    bx, a = boxes[0], accs[0]
    if g.is_empty(bx):
        return
    sh = g.shape(bx) + (a.arr.shape[3],)
    a.store(bx, np.full(sh, F32(p["value"]), dtype=F32).view(U32))


def k_stencil3(p, boxes, accs):
    """C1 (Listing 5 shape): B_i = (0.25*A_{i-1} + 0.5*A_i) + 0.25*A_{i+1},
    clamped indices; acc0 = A read neighborhood(1), acc1 = B write."""
    src, dst = accs
    bx = boxes[1]
    n = g.shape(src.extent)[0]
    i = _ar(bx, 0)
    z = [0]
    xm = src.f32(_clip(i - 1, n), z, z)
    xc = src.f32(i, z, z)
    xp = src.f32(_clip(i + 1, n), z, z)
    out = (F32(0.25) * xm + F32(0.5) * xc) + F32(0.25) * xp
    dst.store(bx, out.view(U32))


def k_wave5(p, boxes, accs):
    """C2 WaveSim 5-point leapfrog ("five-point wave propagation
    stencil"; formula: DESIGN.md reading):
    up = (2*u_c - up) + 0.25*(((u_n + u_s) + (u_w + u_e)) - 4*u_c)."""
    u, up = accs
    bx = boxes[1]
    E = g.shape(u.extent)
    r, c, z = _ar(bx, 0), _ar(bx, 1), [0]
    uc = u.f32(r, c, z)
    un = u.f32(_clip(r - 1, E[0]), c, z)
    us = u.f32(_clip(r + 1, E[0]), c, z)
    uw = u.f32(r, _clip(c - 1, E[1]), z)
    ue = u.f32(r, _clip(c + 1, E[1]), z)
    upc = up.f32(r, c, z)
    lap = ((un + us) + (uw + ue)) - F32(4.0) * uc
    out = (F32(2.0) * uc - upc) + F32(0.25) * lap
    up.store(bx, out.view(U32))


def k_jacobi7(p, boxes, accs):
    """C5 3-D 7-point: b = 0.25*a_c + 0.125*(((a_z- + a_z+) + (a_y- + a_y+)) + (a_x- + a_x+))."""
    a, b = accs
    bx = boxes[1]
    E = g.shape(a.extent)
    z, y, x = _ar(bx, 0), _ar(bx, 1), _ar(bx, 2)
    ac = a.f32(z, y, x)
    zm = a.f32(_clip(z - 1, E[0]), y, x)
    zp = a.f32(_clip(z + 1, E[0]), y, x)
    ym = a.f32(z, _clip(y - 1, E[1]), x)
    yp = a.f32(z, _clip(y + 1, E[1]), x)
    xm = a.f32(z, y, _clip(x - 1, E[2]))
    xp = a.f32(z, y, _clip(x + 1, E[2]))
    out = F32(0.25) * ac + F32(0.125) * (((zm + zp) + (ym + yp)) + (xm + xp))
    b.store(bx, out.view(U32))


NB_DT = F32(2.0 ** -7)
NB_MASS = F32(2.0 ** -20)
NB_EPS2 = F32(2.0 ** -10)


def nbody_accel(P, pi):
    """Sequential sum over j ascending (Listing 1 "timestep"):
    d = p_j - p_i; r2 = ((dx*dx + dy*dy) + dz*dz) + eps2; inv = 1/sqrt(r2);
    s = (inv*inv)*inv; a += d*s.  P: (N,3) float32, pi: (n,3) float32."""
    a = np.zeros(pi.shape, dtype=F32)
    for j in range(P.shape[0]):
        d = P[j][None, :] - pi
        r2 = ((d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1]) + d[:, 2] * d[:, 2]) + NB_EPS2
        inv = F32(1.0) / np.sqrt(r2)
        s = (inv * inv) * inv
        a = a + d * s[:, None]
    return a


def nbody_accel_one(P, pi):
    """Same arithmetic for ONE body, vectorised over j with a sequential
    float32 cumsum (np.cumsum accumulates left to right)."""
    d = P - pi[None, :]
    r2 = ((d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1]) + d[:, 2] * d[:, 2]) + NB_EPS2
    inv = F32(1.0) / np.sqrt(r2)
    s = (inv * inv) * inv
    c = d * s[:, None]
    return np.array([np.cumsum(c[:, k], dtype=F32)[-1] for k in range(3)], dtype=F32)


def k_nbody_step(p, boxes, accs):
    """C3 timestep: acc0 = P read all, acc1 = V read_write one_to_one;
    v += (dt*m)*a."""
    P, V = accs
    bx = boxes[1]
    N = g.shape(P.extent)[0]
    allp = P.f32(np.arange(N), [0], [0])[:, 0, 0, :3]
    i = _ar(bx, 0)
    pi = P.f32(i, [0], [0])[:, 0, 0, :3]
    a = nbody_accel(allp, pi)
    v = V.f32(i, [0], [0]).copy()
    c = NB_DT * NB_MASS
    v[:, 0, 0, :3] = v[:, 0, 0, :3] + c * a
    V.store(bx, v.view(U32))


def k_nbody_update(p, boxes, accs):
    """C3 update: acc0 = V read one_to_one, acc1 = P read_write; p += dt*v."""
    V, P = accs
    bx = boxes[1]
    i = _ar(bx, 0)
    pv = P.f32(i, [0], [0]).copy()
    vv = V.f32(i, [0], [0])
    pv[:, 0, 0, :3] = pv[:, 0, 0, :3] + NB_DT * vv[:, 0, 0, :3]
    P.store(bx, pv.view(U32))


def k_rsim_row(p, boxes, accs):
    """C4 RSim-shaped growth ("appends a new row ... after reading the
    results of all previous time steps"): row t, column i =
    0.5*R[t-1][i] + (0.5/t) * sum_{s<t} R[s][(i+s) mod W], s ascending.
    acc0 = R read fixed [0,t) x [0,W), acc1 = R write remap [t,t+1) x chunk."""
    R, Rw = accs
    bx = boxes[1]
    t = int(p["t"])
    W = g.shape(R.extent)[1]
    cols = _ar(bx, 1)
    acc = np.zeros(cols.shape, dtype=F32)
    for s in range(t):
        acc = acc + R.f32([s], (cols + s) % W, [0])[0, :, 0, 0]
    prev = R.f32([t - 1], cols, [0])[0, :, 0, 0]
    coef = F32(0.5) / F32(t)
    out = F32(0.5) * prev + coef * acc
    Rw.store(bx, out.reshape(g.shape(bx) + (1,)).view(U32))


def _probe_sum(acc, mapper, x, sh):
    """u32 wrapping sum over the element set the read mapper names for element x."""
    kind = mapper[0]
    E = acc.extent
    if kind in ("one_to_one",) or kind == "rw":
        return acc.gather(x[0], x[1], x[2])[..., 0]
    if kind == "all":
        return np.full(sh, U32(int(acc.view_box(E).astype(np.uint64).sum()) & 0xFFFFFFFF), dtype=U32)
    if kind == "fixed":
        bx = mapper[1]
        return np.full(sh, U32(int(acc.view_box(bx).astype(np.uint64).sum()) & 0xFFFFFFFF), dtype=U32)
    if kind == "neighborhood":
        b = mapper[1]
        tot = np.zeros(sh, dtype=U32)
        with np.errstate(over="ignore"):
            for o0 in range(-b[0], b[0] + 1):
                for o1 in range(-b[1], b[1] + 1):
                    for o2 in range(-b[2], b[2] + 1):
                        y0, y1, y2 = x[0] + o0, x[1] + o1, x[2] + o2
                        ok = ((y0 >= E[0][0]) & (y0 < E[1][0]))[:, None, None] & \
                             ((y1 >= E[0][1]) & (y1 < E[1][1]))[None, :, None] & \
                             ((y2 >= E[0][2]) & (y2 < E[1][2]))[None, None, :]
                        v = acc.gather(np.clip(y0, E[0][0], E[1][0] - 1), np.clip(y1, E[0][1], E[1][1] - 1),
                                       np.clip(y2, E[0][2], E[1][2] - 1))[..., 0]
                        tot = tot + np.where(ok, v, U32(0))
        return tot
    raise ValueError(kind)


def k_probe(p, boxes, accs, accesses):
    """Integer coherence probe (u32, order-dependent mixing):
    for write access w and element x of its region:
      h = fmix32((salt + w) ^ fmix32(lin(x)));  for each read access i in
      order: h = fmix32(h ^ S_i(x)), S_i = wrapping u32 sum over the element
      set access i's mapper names for x (read_write: the element x itself)."""
    salt = int(p["salt"])
    outs = []
    for w, (bid, mode, mapper) in enumerate(accesses):
        if mode not in ("write", "read_write"):
            continue
        bx = boxes[w]
        if g.is_empty(bx):
            continue
        E = g.shape(accs[w].extent)
        x = (_ar(bx, 0), _ar(bx, 1), _ar(bx, 2))
        sh = g.shape(bx)
        lin = ((x[0][:, None, None] * E[1]) + x[1][None, :, None]) * E[2] + x[2][None, None, :]
        with np.errstate(over="ignore"):
            h = fmix32((U32((salt + w) & 0xFFFFFFFF)) ^ fmix32((lin & 0xFFFFFFFF).astype(U32)))
            for i, (bid2, mode2, mapper2) in enumerate(accesses):
                if mode2 not in ("read", "read_write"):
                    continue
                S = _probe_sum(accs[i], ("rw",) if mode2 == "read_write" else mapper2, x, sh)
                h = fmix32(h ^ S)
        outs.append((w, bx, h))
    for w, bx, h in outs:
        accs[w].store(bx, h[..., None])


KERNELS = {
    "fill_hash": k_fill_hash,
    "fill_const": k_fill_const,
    "stencil3": k_stencil3,
    "wave5": k_wave5,
    "jacobi7": k_jacobi7,
    "nbody_step": k_nbody_step,
    "nbody_update": k_nbody_update,
    "rsim_row": k_rsim_row,
}


def run_kernel(spec, boxes, accs):
    """Execute task `spec`'s kernel for one chunk: boxes[i] = access i's mapped
    box for the chunk, accs[i] = its accessor."""
    name = spec["kernel"]
    if name == "probe":
        # the probe reads every input before writing any output
        k_probe(spec.get("params", {}), boxes, accs, spec["accesses"])
        return
    KERNELS[name](spec.get("params", {}), boxes, accs)
