"""Work split and range mappers (test infrastructure; oracle).

P:L319-326 (§3.1 Hierarchical Work Assignment): the kernel index space is
split "statically ... along one or more axes"; for the IDAG the command's
index space is split "a second time" over the local devices.  On one node
that is a single split over G devices.

R4 [reading]  1D: along dim 0, part k gets q+1 elements if k < r else q
    (q, r = divmod(len, n)); contiguous in k order.
    2D: G = a*b, a >= b, a-b minimal; a parts along dim 0, b along dim 1;
    device d = i*b + j.  Empty chunks are returned as EMPTY (no kernel).

R5  Range mappers: one_to_one -> chunk (error if not
    inside the extent); neighborhood(b) -> chunk inflated by b per dim,
    clamped to the extent (box inflation incl. corners; "one-
    neighborhood"); all -> extent ("always spans the entire buffer range",
    P:L163); fixed(box) -> box (error if outside); remap(box, kdims)
    [reading, for RSim P:L632]: buffer dim k takes the chunk's interval in
    kernel dim kdims[k], or box's interval when kdims[k] == -1;
    neighborhood_axes(b) [SURVEY NEXT-3] -> the cross: the chunk inflated by
    b[d] along one dim d at a time (mapper_region); its box is the bbox.
"""

from . import geometry as g


class CelError(Exception):
    """Mirrors the C-ABI error convention."""

    INVALID = -1
    OUT_OF_BOUNDS = -2
    OVERLAPPING_WRITE = -3
    STATE = -7

    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


def split_1d(rng, n, dim=0):
    """R4 1D split of box `rng` into n parts along `dim` (EMPTY parts kept)."""
    lo, hi = rng[0][dim], rng[1][dim]
    length = max(0, hi - lo)
    q, r = divmod(length, n)
    out = []
    start = lo
    for k in range(n):
        size = q + (1 if k < r else 0)
        b = g._with_dim(rng, dim, start, start + size)
        out.append(g.EMPTY if g.is_empty(b) else b)
        start += size
    return out


def factor_2d(n):
    """G = a*b with a >= b and a-b minimal (R4): 8->(4,2), 4->(2,2), 2->(2,1)."""
    b = 1
    for c in range(1, n + 1):
        if c * c > n:
            break
        if n % c == 0:
            b = c
    return n // b, b


def split_2d(rng, n):
    a, b = factor_2d(n)
    rows = split_1d(rng, a, 0)
    out = []
    for i in range(a):
        if g.is_empty(rows[i]):
            out.extend([g.EMPTY] * b)
            continue
        cols = split_1d(rows[i], b, 1)
        out.extend(cols)
    return out


def split(rng, n, kind):
    if g.is_empty(rng):
        return [g.EMPTY] * n
    if kind == "1d":
        return split_1d(rng, n)
    if kind == "2d":
        return split_2d(rng, n)
    raise CelError(CelError.INVALID, "unknown split %r" % (kind,))


def apply_mapper(mapper, chunk, extent):
    """R5: kernel chunk -> buffer box."""
    kind = mapper[0]
    if g.is_empty(chunk):
        return g.EMPTY
    if kind == "one_to_one":
        if not g.box_contains(extent, chunk):
            raise CelError(CelError.OUT_OF_BOUNDS, "one_to_one chunk outside buffer extent")
        return chunk
    if kind == "neighborhood":
        border = tuple(mapper[1]) + (0,) * (3 - len(mapper[1]))
        mn = tuple(chunk[0][d] - border[d] for d in range(3))
        mx = tuple(chunk[1][d] + border[d] for d in range(3))
        return g.box_intersect((mn, mx), extent)
    if kind == "neighborhood_axes":
        # the bounding box of the cross (mapper_region is the region itself)
        border = tuple(mapper[1]) + (0,) * (3 - len(mapper[1]))
        mn = tuple(chunk[0][d] - border[d] for d in range(3))
        mx = tuple(chunk[1][d] + border[d] for d in range(3))
        return g.box_intersect((mn, mx), extent)
    if kind == "all":
        return extent
    if kind == "fixed":
        b = mapper[1]
        if not g.box_contains(extent, b):
            raise CelError(CelError.OUT_OF_BOUNDS, "fixed box outside buffer extent")
        return b
    if kind == "remap":
        fixed, kdims = mapper[1], mapper[2]
        mn, mx = [], []
        for k in range(3):
            src = kdims[k]
            if src >= 0:
                mn.append(chunk[0][src])
                mx.append(chunk[1][src])
            else:
                mn.append(fixed[0][k])
                mx.append(fixed[1][k])
        b = (tuple(mn), tuple(mx))
        if g.is_empty(b):
            return g.EMPTY
        if not g.box_contains(extent, b):
            raise CelError(CelError.OUT_OF_BOUNDS, "remap box outside buffer extent")
        return b
    raise CelError(CelError.INVALID, "unknown mapper %r" % (kind,))


def mapper_region(mapper, chunk, extent):
    """R5 / SURVEY NEXT-3: the buffer region a chunk accesses.  Equal to the
    mapper's box for every kind except `neighborhood_axes`, the axis-only
    neighbourhood (a stencil that reads no corners): the union over dims d of
    the chunk inflated by border[d] in dim d alone, clamped to the extent."""
    if mapper[0] != "neighborhood_axes":
        bx = apply_mapper(mapper, chunk, extent)
        return () if g.is_empty(bx) else (bx,)
    if g.is_empty(chunk):
        return ()
    border = tuple(mapper[1]) + (0,) * (3 - len(mapper[1]))
    parts = [chunk]
    for d in range(3):
        if border[d] > 0:
            parts.append(g._with_dim(chunk, d, chunk[0][d] - border[d], chunk[1][d] + border[d]))
    return g.region_intersect(g.region_union(*[(p,) for p in parts]), (extent,))


READS = ("read", "read_write")
WRITES = ("write", "read_write")
