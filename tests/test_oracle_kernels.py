"""Pins for oracle/kernels.py: published test vectors, closed forms, special
cases and an independent float64 evaluation (catches dropped terms, wrong
signs, swapped operands)."""

import numpy as np

from oracle import geometry as g
from oracle import kernels as K

F32 = np.float32


def acc_of(arr32, extent):
    """Wrap a float32/uint32 ndarray of shape extent(+words) as a full-extent accessor."""
    ext = g.box([0] * len(extent), list(extent))
    a = np.ascontiguousarray(arr32).view(np.uint32).reshape(g.shape(ext) + (-1,))
    return K.Acc(a.copy(), ext, ext), ext


def test_splitmix64_reference_vector():
    # Vigna's splitmix64.c seeded with x = 0: first outputs
    assert int(K.splitmix64(np.uint64(0))) == 0xE220A8397B1DCDAF
    assert int(K.splitmix64(np.uint64(0x9E3779B97F4A7C15))) == 0x6E789E6AA1B965F4


def test_init_value_range_and_exactness():
    v = K.init_value(1, np.arange(1 << 16, dtype=np.uint64))
    assert v.dtype == np.float32
    assert (v >= -1).all() and (v < 1).all()
    # exact multiples of 2^-23 (24-bit integer scaled, then 2x-1 exactly)
    q = v.astype(np.float64) * 2 ** 23
    assert (q == np.round(q)).all()
    # equals the float64 evaluation of the definition
    h = K.splitmix64(np.uint64(1) + np.arange(1 << 16, dtype=np.uint64))
    ref = 2.0 * ((h >> np.uint64(40)).astype(np.float64) / 2 ** 24) - 1.0
    assert (v.astype(np.float64) == ref).all()


def test_fmix32_bijective_sample():
    x = np.arange(1 << 18, dtype=np.uint32) * np.uint32(2654435761)
    assert len(np.unique(K.fmix32(x))) == len(np.unique(x))
    assert int(K.fmix32(np.uint32(0))) == 0


def test_wave5_constant_field_invariant():
    c = F32(0.375)
    u, ext = acc_of(np.full((9, 7), c, dtype=F32), (9, 7))
    up, _ = acc_of(np.full((9, 7), c, dtype=F32), (9, 7))
    K.k_wave5({}, [ext, ext], [u, up])
    assert (up.arr.view(F32) == c).all()


def test_wave5_linear_ramp_interior():
    # interior Laplacian of a linear ramp is exactly 0 -> up' = 2u - up = u when up = u
    i, j = np.meshgrid(np.arange(10), np.arange(12), indexing="ij")
    f = (F32(0.125) * i + F32(0.0625) * j).astype(F32)
    u, ext = acc_of(f, (10, 12))
    up, _ = acc_of(f, (10, 12))
    K.k_wave5({}, [ext, ext], [u, up])
    out = up.arr.view(F32)[..., 0, 0]
    assert (out[1:-1, 1:-1] == f[1:-1, 1:-1]).all()


def test_wave5_vs_float64():
    r = np.random.default_rng(0)
    u0 = r.uniform(-1, 1, (13, 11)).astype(F32)
    p0 = r.uniform(-1, 1, (13, 11)).astype(F32)
    u, ext = acc_of(u0, (13, 11))
    up, _ = acc_of(p0, (13, 11))
    K.k_wave5({}, [ext, ext], [u, up])
    U = np.pad(u0.astype(np.float64), 1, mode="edge")
    lap = U[:-2, 1:-1] + U[2:, 1:-1] + U[1:-1, :-2] + U[1:-1, 2:] - 4 * U[1:-1, 1:-1]
    ref = 2 * u0 - p0.astype(np.float64) + 0.25 * lap
    assert np.allclose(up.arr.view(F32)[..., 0, 0], ref, atol=1e-6, rtol=0)


def test_jacobi7_constant_and_float64():
    a, ext = acc_of(np.full((5, 6, 7), F32(-0.75), dtype=F32), (5, 6, 7))
    b, _ = acc_of(np.zeros((5, 6, 7), dtype=F32), (5, 6, 7))
    K.k_jacobi7({}, [ext, ext], [a, b])
    assert (b.arr.view(F32) == F32(-0.75)).all()         # weights sum to exactly 1
    r = np.random.default_rng(1)
    x = r.uniform(-1, 1, (5, 6, 7)).astype(F32)
    a, ext = acc_of(x, (5, 6, 7))
    K.k_jacobi7({}, [ext, ext], [a, b])
    X = np.pad(x.astype(np.float64), 1, mode="edge")
    ref = 0.25 * X[1:-1, 1:-1, 1:-1] + 0.125 * (X[:-2, 1:-1, 1:-1] + X[2:, 1:-1, 1:-1] + X[1:-1, :-2, 1:-1]
                                                + X[1:-1, 2:, 1:-1] + X[1:-1, 1:-1, :-2] + X[1:-1, 1:-1, 2:])
    assert np.allclose(b.arr.view(F32)[..., 0], ref, atol=1e-6, rtol=0)


def test_stencil3_vs_float64():
    r = np.random.default_rng(2)
    x = r.uniform(-1, 1, 33).astype(F32)
    a, ext = acc_of(x, (33,))
    b, _ = acc_of(np.zeros(33, dtype=F32), (33,))
    K.k_stencil3({}, [ext, ext], [a, b])
    X = np.pad(x.astype(np.float64), 1, mode="edge")
    ref = 0.25 * X[:-2] + 0.5 * X[1:-1] + 0.25 * X[2:]
    assert np.allclose(b.arr.view(F32)[:, 0, 0, 0], ref, atol=1e-7, rtol=0)


def test_nbody_special_cases_and_float64():
    # a single body feels exactly zero force (d = 0 contributes 0)
    one = np.array([[0.3, -0.2, 0.1]], dtype=F32)
    assert (K.nbody_accel(one, one) == 0).all()
    # two symmetric bodies: exactly opposite accelerations
    two = np.array([[0.5, 0.25, -0.125], [-0.5, -0.25, 0.125]], dtype=F32)
    a = K.nbody_accel(two, two)
    assert (a[0] == -a[1]).all() and (a[0] != 0).all()
    # attraction: body 0 accelerates towards body 1
    assert (np.sign(a[0]) == np.sign(two[1] - two[0])).all()
    r = np.random.default_rng(3)
    P = r.uniform(-1, 1, (64, 3)).astype(F32)
    a = K.nbody_accel(P, P)
    d = P[None, :, :].astype(np.float64) - P[:, None, :]
    r2 = (d ** 2).sum(-1) + 2.0 ** -10
    ref = (d / r2[..., None] ** 1.5).sum(1)
    assert np.allclose(a, ref, rtol=1e-4, atol=1e-3)
    # the cumsum evaluation is the same sequential sum, bit for bit
    for i in (0, 17, 63):
        assert (K.nbody_accel_one(P, P[i]) == a[i]).all()


def test_nbody_update_step():
    N = 8
    p = np.zeros((N, 4), dtype=F32)
    v = np.full((N, 4), F32(1.0), dtype=F32)
    P, ext = acc_of(p, (N,))
    V, _ = acc_of(v, (N,))
    K.k_nbody_update({}, [ext, ext], [V, P])
    out = P.arr.view(F32)[:, 0, 0, :]
    assert (out[:, :3] == F32(2.0 ** -7)).all() and (out[:, 3] == 0).all()


def test_rsim_row_constant_and_float64():
    T, W = 6, 10
    R = np.zeros((T, W), dtype=F32)
    R[:3] = F32(0.5)
    acc, ext = acc_of(R, (T, W))
    wbox = g.box([3, 0], [4, W])
    K.k_rsim_row({"t": 3}, [g.box([0, 0], [3, W]), wbox], [acc, acc])
    row = acc.arr.view(F32)[3, :, 0, 0]
    assert np.allclose(row, 0.5, atol=1e-7)
    r = np.random.default_rng(4)
    R = r.uniform(-1, 1, (T, W)).astype(F32)
    acc, ext = acc_of(R, (T, W))
    K.k_rsim_row({"t": 5}, [g.box([0, 0], [5, W]), g.box([5, 0], [6, W])], [acc, acc])
    ref = np.array([0.5 * R[4, i] + 0.5 / 5 * sum(R[s, (i + s) % W] for s in range(5)) for i in range(W)])
    assert np.allclose(acc.arr.view(F32)[5, :, 0, 0], ref, atol=1e-6)


def test_probe_is_sensitive_to_every_read_element():
    n = 12
    ext = g.box([0], [n])
    base = np.arange(n, dtype=np.uint32) * np.uint32(7)
    spec = {"kernel": "probe", "params": {"salt": 5},
            "accesses": [(1, "write", ("one_to_one",)), (0, "read", ("neighborhood", (1, 0, 0)))]}

    def out(src):
        a = K.Acc(src.reshape(n, 1, 1, 1).copy(), ext, ext)
        o = K.Acc(np.zeros((n, 1, 1, 1), dtype=np.uint32), ext, ext)
        K.run_kernel(spec, [ext, ext], [o, a])
        return o.arr[:, 0, 0, 0]

    ref = out(base)
    for k in range(n):
        m = base.copy()
        m[k] ^= np.uint32(1 << 9)
        diff = np.nonzero(out(m) != ref)[0]
        assert set(diff) == {i for i in (k - 1, k, k + 1) if 0 <= i < n}
