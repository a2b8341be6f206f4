"""Box / Region / RegionMap — the oracle's integer set algebra (test infrastructure).

Paper basis: buffers are tracked in "rectangular regions" (§3.4) and
"subregions" that are "locally up-to-date on what memory ids" (P:L371-372,
§3.3).  The paper does not fix a representation; readings R1-R3:

R1  A Box is half-open [min, max) in 3 dims; dims beyond the buffer's are
    [0,1).  Dim 0 is the slowest (row-major).  There is one empty box EMPTY.
R2  A Region is a tuple of disjoint boxes in *maximal-slab canonical form*:
    dim 0 is cut exactly where the (dim1, dim2) cross-section changes; each
    slab's cross-section is canonical recursively (1-D: merged intervals);
    boxes come out sorted lexicographically by min.  Equal point sets give
    identical tuples.
R3  A RegionMap is a total map extent -> value, stored as value -> Region;
    query() returns (region, value) pairs sorted by value key.

Everything here is plain Python on tuples; slow, but obviously correct and
checked against a per-element bitmap in tests/test_oracle_geometry.py.
"""

EMPTY = ((0, 0, 0), (0, 0, 0))


def box(mn, mx):
    """Box from 1..3-element min/max sequences; missing dims become [0,1) (R1)."""
    mn = tuple(int(v) for v in mn) + (0,) * (3 - len(mn))
    mx = tuple(int(v) for v in mx) + (1,) * (3 - len(mx))
    b = (mn, mx)
    return EMPTY if is_empty(b) else b


def is_empty(b):
    return any(b[1][d] <= b[0][d] for d in range(3))


def volume(b):
    if is_empty(b):
        return 0
    v = 1
    for d in range(3):
        v *= b[1][d] - b[0][d]
    return v


def shape(b):
    return tuple(b[1][d] - b[0][d] for d in range(3))


def box_intersect(a, b):
    mn = tuple(max(a[0][d], b[0][d]) for d in range(3))
    mx = tuple(min(a[1][d], b[1][d]) for d in range(3))
    r = (mn, mx)
    return EMPTY if is_empty(r) else r


def box_contains(outer, inner):
    """inner ⊆ outer (every set contains the empty box)."""
    if is_empty(inner):
        return True
    if is_empty(outer):
        return False
    return all(outer[0][d] <= inner[0][d] and inner[1][d] <= outer[1][d] for d in range(3))


def bounding_box(boxes):
    """Smallest box containing all given boxes; EMPTY for none (SPEC bounding_box)."""
    bs = [b for b in boxes if not is_empty(b)]
    if not bs:
        return EMPTY
    mn = tuple(min(b[0][d] for b in bs) for d in range(3))
    mx = tuple(max(b[1][d] for b in bs) for d in range(3))
    return (mn, mx)


def _with_dim(b, d, lo, hi):
    mn = list(b[0])
    mx = list(b[1])
    mn[d] = lo
    mx[d] = hi
    return (tuple(mn), tuple(mx))


def box_subtract(a, b):
    """a minus b as a list of disjoint boxes (peel slabs off dim 0, then 1, then 2)."""
    i = box_intersect(a, b)
    if is_empty(i):
        return [] if is_empty(a) else [a]
    out = []
    cur = a
    for d in range(3):
        if cur[0][d] < i[0][d]:
            out.append(_with_dim(cur, d, cur[0][d], i[0][d]))
        if i[1][d] < cur[1][d]:
            out.append(_with_dim(cur, d, i[1][d], cur[1][d]))
        cur = _with_dim(cur, d, i[0][d], i[1][d])
    return out


def _canon(bs, d):
    """Canonical boxes of the union of `bs` (non-empty, possibly overlapping) over
    dims d..2.  All boxes in `bs` agree on dims < d (the caller projected them)."""
    if d == 2:
        ivs = sorted((b[0][2], b[1][2]) for b in bs)
        merged = []
        for lo, hi in ivs:
            if merged and lo <= merged[-1][1]:
                if hi > merged[-1][1]:
                    merged[-1][1] = hi
            else:
                merged.append([lo, hi])
        proto = bs[0]
        return [_with_dim(proto, 2, lo, hi) for lo, hi in merged]
    cuts = sorted({c for b in bs for c in (b[0][d], b[1][d])})
    slabs = []
    for lo, hi in zip(cuts, cuts[1:]):
        cover = [_with_dim(b, d, 0, 1) for b in bs if b[0][d] <= lo and hi <= b[1][d]]
        if not cover:
            continue
        sub = tuple(_canon(cover, d + 1))
        if slabs and slabs[-1][1] == lo and slabs[-1][2] == sub:
            slabs[-1][1] = hi
        else:
            slabs.append([lo, hi, sub])
    out = []
    for lo, hi, sub in slabs:
        for sb in sub:
            out.append(_with_dim(sb, d, lo, hi))
    return out


def canon(boxes):
    """Region (R2 canonical form) of the union of arbitrary boxes."""
    bs = [b for b in boxes if not is_empty(b)]
    if not bs:
        return ()
    return tuple(_canon(bs, 0))


def region(*boxes):
    return canon(boxes)


def region_union(*regions):
    return canon([b for r in regions for b in r])


def region_intersect(a, b):
    return canon([box_intersect(x, y) for x in a for y in b])


def region_difference(a, b):
    out = list(a)
    for y in b:
        nxt = []
        for x in out:
            nxt.extend(box_subtract(x, y))
        out = nxt
        if not out:
            break
    return canon(out)


def region_volume(r):
    return sum(volume(b) for b in r)


def region_bbox(r):
    return bounding_box(r)


def _key(v):
    if isinstance(v, frozenset):
        return (1, tuple(sorted(v)))
    return (0, v)


class RegionMap:
    """Total map from every point of `extent` to a value (R3; SPEC RegionMap).

    Stored as {value: canonical Region}; regions of distinct values partition
    the extent.  Equal values are merged by construction, so the entry count is
    bounded by the number of distinct live values."""

    def __init__(self, extent, default):
        self.extent = extent
        self.m = {default: (extent,)} if not is_empty(extent) else {}

    def copy(self):
        c = RegionMap.__new__(RegionMap)
        c.extent = self.extent
        c.m = dict(self.m)
        return c

    def update(self, reg, value):
        """Overwrite exactly `reg` (⊆ extent) with `value`."""
        reg = region_intersect(reg, (self.extent,))
        if not reg:
            return
        new = {}
        for v, r in self.m.items():
            rr = region_difference(r, reg)
            if rr:
                new[v] = rr
        new[value] = region_union(new.get(value, ()), reg)
        self.m = new

    def apply(self, reg, fn):
        """Replace value v by fn(v) on `reg` only."""
        reg = region_intersect(reg, (self.extent,))
        if not reg:
            return
        new = {}
        for v, r in self.m.items():
            inside = region_intersect(r, reg)
            outside = region_difference(r, reg) if inside else r
            if outside:
                new[v] = region_union(new.get(v, ()), outside)
            if inside:
                nv = fn(v)
                new[nv] = region_union(new.get(nv, ()), inside)
        self.m = new

    def map_values(self, fn):
        """Replace every value v by fn(v) everywhere, merging equal results."""
        new = {}
        for v, r in self.m.items():
            nv = fn(v)
            new[nv] = region_union(new.get(nv, ()), r)
        self.m = new

    def query(self, reg):
        """Partition of `reg` by value: [(region, value)] sorted by value key."""
        out = []
        for v, r in self.m.items():
            i = region_intersect(r, reg)
            if i:
                out.append((i, v))
        out.sort(key=lambda p: _key(p[1]))
        return out

    def region_where(self, pred):
        return region_union(*[r for v, r in self.m.items() if pred(v)])

    def values(self):
        return sorted(self.m.keys(), key=_key)

    def lookup(self, point):
        p = tuple(point) + (0,) * (3 - len(point))
        for v, r in self.m.items():
            for b in r:
                if all(b[0][d] <= p[d] < b[1][d] for d in range(3)):
                    return v
        raise KeyError(point)
