"""Pins for oracle/geometry.py against a per-element bitmap
and the SPEC worked examples."""

import random

import numpy as np
import pytest

from oracle import geometry as g

B = g.box


def bitmap(region, n=(8, 8, 8)):
    m = np.zeros(n, dtype=bool)
    for b in region:
        m[b[0][0]:b[1][0], b[0][1]:b[1][1], b[0][2]:b[1][2]] = True
    return m


def rand_box(r, n=(8, 8, 8), dims=3):
    mn, mx = [], []
    for d in range(dims):
        a = r.randrange(0, n[d])
        c = r.randrange(a, n[d] + 1)
        mn.append(a)
        mx.append(c)
    return B(mn, mx)


def rand_region(r, k, dims=3):
    return g.canon([rand_box(r, dims=dims) for _ in range(k)])


def test_spec_examples():
    # S:L52-53
    assert g.box_intersect(B([0], [8]), B([4], [12])) == B([4], [8])
    assert g.is_empty(g.box_intersect(B([0], [8]), B([8], [12])))
    # S:L61-62
    assert g.region_union(g.region(B([0], [4])), g.region(B([4], [8]))) == g.region(B([0], [8]))
    assert g.region_difference(g.region(B([0], [8])), g.region(B([0], [8]))) == ()
    # S:L70-71
    assert g.bounding_box(g.region(B([0], [2]), B([6], [8]))) == B([0], [8])
    assert g.bounding_box(g.region(B([3], [5]))) == B([3], [5])
    # S:L79-81
    m = g.RegionMap(B([0], [12]), "U")
    m.update(g.region(B([0], [8])), "A")
    assert m.query(g.region(B([2], [4]))) == [(g.region(B([2], [4])), "A")]
    m.update(g.region(B([4], [12])), "B")
    assert m.query(g.region(B([0], [12]))) == [(g.region(B([0], [4])), "A"), (g.region(B([4], [12])), "B")]
    assert m.query(()) == []


def test_empty_box_is_unique():
    assert B([3], [3]) == g.EMPTY
    assert B([0, 5], [4, 2]) == g.EMPTY
    assert g.canon([g.EMPTY, B([1], [1])]) == ()


def test_canonical_form_shape():
    # an L-shape: maximal slabs along dim 0 (R2)
    r = g.region(B([0, 0], [2, 4]), B([2, 0], [4, 2]))
    assert r == (B([0, 0], [2, 4]), B([2, 0], [4, 2]))
    # the same point set from another decomposition
    r2 = g.region(B([0, 0], [4, 2]), B([0, 2], [2, 4]))
    assert r == r2
    # sorted lexicographically by min, pairwise disjoint
    for x, y in zip(r, r[1:]):
        assert x[0] < y[0]


@pytest.mark.parametrize("op", ["union", "intersect", "difference"])
def test_region_ops_vs_bitmap(op):
    r = random.Random({"union": 1, "intersect": 2, "difference": 3}[op])
    for _ in range(1500):
        a = rand_region(r, r.randrange(0, 4))
        b = rand_region(r, r.randrange(0, 4))
        if op == "union":
            res, exp = g.region_union(a, b), bitmap(a) | bitmap(b)
        elif op == "intersect":
            res, exp = g.region_intersect(a, b), bitmap(a) & bitmap(b)
        else:
            res, exp = g.region_difference(a, b), bitmap(a) & ~bitmap(b)
        assert (bitmap(res) == exp).all()
        # disjoint boxes, volume matches the bitmap
        assert g.region_volume(res) == int(exp.sum())
        # canonical: re-deriving from the bitmap's unit cells gives the same tuple
        cells = [B(p, [p[0] + 1, p[1] + 1, p[2] + 1]) for p in zip(*np.nonzero(exp))]
        assert g.canon(cells) == res


def test_bbox_vs_bitmap():
    r = random.Random(4)
    for _ in range(1000):
        a = rand_region(r, r.randrange(0, 4))
        bb = g.bounding_box(a)
        m = bitmap(a)
        if not m.any():
            assert bb == g.EMPTY
            continue
        idx = np.nonzero(m)
        assert bb == B([int(i.min()) for i in idx], [int(i.max()) + 1 for i in idx])


def test_canonicity_under_resplitting():
    r = random.Random(5)
    for _ in range(300):
        boxes = [rand_box(r) for _ in range(r.randrange(1, 5))]
        ref = g.canon(boxes)
        # shuffle, and re-split every box at a random cut
        pieces = []
        for b in boxes:
            d = r.randrange(3)
            if b[1][d] - b[0][d] >= 2:
                c = r.randrange(b[0][d] + 1, b[1][d])
                pieces += [g._with_dim(b, d, b[0][d], c), g._with_dim(b, d, c, b[1][d])]
            else:
                pieces.append(b)
        r.shuffle(pieces)
        assert g.canon(pieces) == ref


def test_regionmap_vs_pointwise_and_bounded():
    r = random.Random(6)
    ext = B([0, 0, 0], [8, 8, 8])
    m = g.RegionMap(ext, -1)
    ref = np.full((8, 8, 8), -1)
    for k in range(200):
        reg = rand_region(r, r.randrange(1, 3))
        v = r.randrange(0, 4)                    # few distinct values
        m.update(reg, v)
        ref[bitmap(reg)] = v
        q = rand_region(r, 2)
        for part, val in m.query(q):
            assert (ref[bitmap(part)] == val).all()
        assert sum(g.region_volume(p) for p, _ in m.query(q)) == int(bitmap(q).sum())
        # entry count bounded by distinct values, not by the extent
        assert len(m.m) <= 5
    # apply() and map_values()
    m2 = m.copy()
    m2.map_values(lambda v: 0 if v < 2 else v)
    for part, val in m2.query((ext,)):
        assert (np.where(ref < 2, 0, ref)[bitmap(part)] == val).all()
