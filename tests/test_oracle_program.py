"""Pins for the work split (R4) and range mappers (R5)."""

import random

import pytest

from oracle import geometry as g
from oracle.program import CelError, apply_mapper, factor_2d, split, split_1d

B = g.box


def test_split_examples():
    N = 1 << 20
    # P:L240 "operates on the first half of the task index space"
    assert split(B([0], [N]), 2, "1d")[0] == B([0], [N // 2])
    # S:L250 remainder to the lower ids
    assert split(B([0], [7]), 2, "1d") == [B([0], [4]), B([4], [7])]
    # S:L251 degenerate oversplit: 4 unit chunks + 4 empty
    s = split(B([0], [4]), 8, "1d")
    assert s[:4] == [B([i], [i + 1]) for i in range(4)] and all(x == g.EMPTY for x in s[4:])


def test_hierarchical_split_gives_quarters():
    # node split in halves, then each half over 2 devices
    N = 1 << 12
    halves = split(B([0], [N]), 2, "1d")
    quarters = [q for h in halves for q in split_1d(h, 2)]
    assert quarters == split(B([0], [N]), 4, "1d")
    assert quarters[0] == B([0], [N // 4])          # "the first quarter"


@pytest.mark.parametrize("n,ab", [(1, (1, 1)), (2, (2, 1)), (3, (3, 1)), (4, (2, 2)), (6, (3, 2)), (8, (4, 2))])
def test_factor_2d(n, ab):
    assert factor_2d(n) == ab


def test_split_properties():
    r = random.Random(7)
    for _ in range(500):
        dims = r.randrange(1, 4)
        ext = [r.randrange(0, 40) for _ in range(dims)]
        rng = B([0] * dims, ext) if all(ext) else g.EMPTY
        n = r.randrange(1, 9)
        kind = "2d" if dims >= 2 and r.random() < 0.5 else "1d"
        parts = split(rng, n, kind)
        assert len(parts) == n
        nonempty = [p for p in parts if p != g.EMPTY]
        # disjoint, union = range
        assert g.canon(nonempty) == (g.canon([rng]) if rng != g.EMPTY else ())
        assert sum(g.volume(p) for p in nonempty) == g.volume(rng)
        if kind == "1d" and rng != g.EMPTY:
            sizes = [p[1][0] - p[0][0] if p != g.EMPTY else 0 for p in parts]
            assert max(sizes) - min(sizes) <= 1
            assert sizes == sorted(sizes, reverse=True)


def test_split_2d_device_order():
    # R4: device d = i*b + j with (a, b) = (4, 2) for 8
    parts = split(B([0, 0, 0], [8, 4, 5]), 8, "2d")
    assert parts[0] == B([0, 0, 0], [2, 2, 5])
    assert parts[1] == B([0, 2, 0], [2, 4, 5])
    assert parts[7] == B([6, 2, 0], [8, 4, 5])


def test_mapper_examples():
    ext = B([0], [1024])
    ch = B([0], [512])
    assert apply_mapper(("one_to_one",), ch, ext) == B([0], [512])
    assert apply_mapper(("all",), ch, ext) == ext
    assert apply_mapper(("neighborhood", (1, 0, 0)), B([4], [8]), B([0], [16])) == B([3], [9])
    # clamped at the extent
    assert apply_mapper(("neighborhood", (1, 0, 0)), B([0], [8]), B([0], [16])) == B([0], [9])
    # box inflation includes corners (R5 reading)
    assert apply_mapper(("neighborhood", (1, 1, 0)), B([2, 2], [4, 4]), B([0, 0], [8, 8])) == B([1, 1], [5, 5])
    # remap: 1-D kernel writing one row of a 2-D buffer (RSim, R5)
    assert apply_mapper(("remap", ((5, 0, 0), (6, 1, 1)), (-1, 0, -1)), B([10], [20]),
                        B([0, 0], [8, 100])) == B([5, 10], [6, 20])


def test_mapper_errors():
    with pytest.raises(CelError) as e:
        apply_mapper(("one_to_one",), B([0], [20]), B([0], [16]))
    assert e.value.code == CelError.OUT_OF_BOUNDS
    with pytest.raises(CelError):
        apply_mapper(("fixed", B([10], [20])), B([0], [4]), B([0], [16]))


def test_mapper_monotone():
    # chunk1 ⊆ chunk2 ⇒ mapped(chunk1) ⊆ mapped(chunk2); all/fixed constant
    r = random.Random(8)
    ext = B([0, 0, 0], [16, 16, 16])
    for _ in range(500):
        c2 = B([r.randrange(0, 8) for _ in range(3)], [r.randrange(8, 17) for _ in range(3)])
        c1 = B([r.randrange(c2[0][d], c2[1][d]) for d in range(3)], [c2[1][d] for d in range(3)])
        for mp in [("one_to_one",), ("neighborhood", (1, 2, 0)), ("all",), ("fixed", B([1, 1, 1], [3, 3, 3]))]:
            assert g.box_contains(apply_mapper(mp, c2, ext), apply_mapper(mp, c1, ext))


def test_axis_neighborhood_region():
    """The axis-only neighbourhood is the union of the chunk
    inflated along each dimension alone: a cross; volume by inclusion-exclusion,
    and brute force on a small grid."""
    from oracle.program import mapper_region
    ext = g.box([0, 0], [10, 10])
    ch = g.box([2, 3], [5, 7])
    r = mapper_region(("neighborhood_axes", (1, 1, 0)), ch, ext)
    assert g.region_volume(r) == 5 * 4 + 3 * 6 - 3 * 4
    pts = {(z, y) for z in range(10) for y in range(10)
           if (2 <= z < 5 and 2 <= y < 8) or (1 <= z < 6 and 3 <= y < 7)}
    got = {(z, y) for b in r for z in range(b[0][0], b[1][0]) for y in range(b[0][1], b[1][1])}
    assert got == pts
    # clamped at the extent, and equal to the box mapper in 1-D
    r0 = mapper_region(("neighborhood_axes", (2, 2, 0)), g.box([0, 0], [3, 3]), ext)
    assert g.region_bbox(r0) == g.box([0, 0], [5, 5]) and g.region_volume(r0) == 9 + 2 * 6
    assert mapper_region(("neighborhood_axes", (1, 0, 0)), g.box([3], [5]), g.box([0], [9])) == \
        mapper_region(("neighborhood", (1, 0, 0)), g.box([3], [5]), g.box([0], [9]))
