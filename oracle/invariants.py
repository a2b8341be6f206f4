"""Brute-force invariant checker for an instruction log (test infrastructure).

Implements the checks SURVEY §8(c) / north_star name, per element, on tiny
buffers, for ANY instruction log (the oracle's or the C++ scheduler's):

  * topological ids: every dependency has a smaller iid;
  * allocation lifetime: every use of an allocation is a descendant of its
    alloc and an ancestor of its free; nothing uses it after the free
    (Fig. 4 legend "allocation lifetime");
  * hazards: for every (allocation, element), the previous writer is an
    ancestor of every later reader (RAW) and writer (WAW), and every reader
    since the last write is an ancestor of the next writer (WAR) — "no
    write-after-read hazard is left unordered" (north_star);
  * coverage: every element a kernel (or readback) reads carries exactly
    the value of the buffer's last writer in task order ("every read is
    covered by exactly one up-to-date last writer", north_star);
  * allocation shape (R9, SURVEY §8(c) pin table), per (buffer, memory):
    - non-overlap: "buffer backing allocations remain non-overlapping"
       — outside a resize chain (alloc, resize copies, free)
      the live allocations are pairwise disjoint;
    - never shrink: "we never emit instructions to downsize a buffer
      allocation" — an alloc that overlaps a live allocation
      contains it (it replaces it), a resize copy goes into an allocation
      containing its source, and a free that is not the buffer's last
      reference leaves a live allocation containing the freed box;
    - pairing: every alloc has exactly one free, and none is live after
      shutdown ("all allocations are however returned back to the system
      eventually").

Values are symbolic tokens (the producing kernel's iid), not bytes.
"""

import numpy as np

from . import geometry as g
from .program import mapper_region, READS, WRITES
from .scheduler import HOST_AID, USER_AID, _norm_mapper


class InvariantError(AssertionError):
    pass


def _tobox(jb):
    return (tuple(jb[0]), tuple(jb[1]))


def _sl(abox, bx):
    b = abox[0]
    return (slice(bx[0][0] - b[0], bx[1][0] - b[0]), slice(bx[0][1] - b[1], bx[1][1] - b[1]),
            slice(bx[0][2] - b[2], bx[1][2] - b[2]))


class _A:
    def __init__(self, box, alloc_iid, host=False):
        sh = g.shape(box)
        self.box = box
        self.alloc_iid = alloc_iid
        self.writer = np.full(sh, -1, dtype=np.int64)
        self.token = np.full(sh, -2, dtype=np.int64)       # -2 garbage
        self.readers = []                                   # [(iid, bool mask)]
        self.freed = None
        if host:
            self.token[...] = -1                            # host-initialised data


def check_allocations(log, closed=True):
    """R9 allocation shape on any log: see the
    module docstring.  `closed`: the log ends after shutdown, so nothing may
    still be live."""
    buf_of = {}
    last_use = {}                     # buffer -> index of its last non-free reference
    for i, rec in enumerate(log):
        k = rec["kind"]
        if k == "alloc":
            buf_of[rec["aid"]] = rec["buffer"]
        if k in ("alloc", "copy", "send", "receive", "split_receive", "await_receive"):
            last_use[rec["buffer"]] = i
        elif k == "kernel":
            for aid in rec["bindings"]:
                if aid in buf_of:
                    last_use[buf_of[aid]] = i
    live = {}                         # (buffer, mem) -> {aid: box}
    where = {}                        # aid -> (buffer, mem)
    freed = set()
    dirty = False                     # a resize chain may be open: disjointness re-checked after it
    for i, rec in enumerate(log):
        k = rec["kind"]
        in_chain = k in ("alloc", "free") or (k == "copy" and rec["reason"] == "resize")
        if dirty and not in_chain:
            for key, d in live.items():
                items = sorted(d.items())
                for x in range(len(items)):
                    for y in range(x + 1, len(items)):
                        if not g.is_empty(g.box_intersect(items[x][1], items[y][1])):
                            raise InvariantError("allocations %d and %d of buffer %d on M%d overlap at instruction %d "
                                                 "(P:L350)" % (items[x][0], items[y][0], key[0], key[1], i))
            dirty = False
        if k == "alloc":
            aid, key, bx = rec["aid"], (rec["buffer"], rec["mem"]), _tobox(rec["box"])
            if aid in where or aid in freed:
                raise InvariantError("allocation %d allocated twice (S:L376)" % aid)
            for o, ob in live.get(key, {}).items():
                if not g.is_empty(g.box_intersect(ob, bx)) and not g.box_contains(bx, ob):
                    raise InvariantError("alloc %d overlaps live allocation %d without containing it "
                                         "(downsize / overlap, P:L350, P:L364)" % (aid, o))
            live.setdefault(key, {})[aid] = bx
            where[aid] = key
            dirty = True
        elif k == "copy" and rec["reason"] == "resize":
            s, d = rec["src_aid"], rec["dst_aid"]
            if s in where and d in where and not g.box_contains(live[where[d]][d], live[where[s]][s]):
                raise InvariantError("resize copy %d: destination allocation %d does not contain source %d (P:L364)"
                                     % (i, d, s))
        elif k == "free":
            aid = rec["aid"]
            if aid not in where:
                raise InvariantError("free %d of allocation %d that is not live (S:L376)" % (i, aid))
            key = where.pop(aid)
            bx = live[key].pop(aid)
            freed.add(aid)
            if last_use.get(key[0], -1) > i and not any(g.box_contains(ob, bx) for ob in live[key].values()):
                raise InvariantError("free %d drops allocation %d of buffer %d before its last use with no live "
                                     "allocation containing it (downsize, P:L364)" % (i, aid, key[0]))
    if closed:
        left = sorted(where)
        if left:
            raise InvariantError("allocations %s are never freed (P:L365, S:L376)" % left)
    return {"allocs": len(where) + len(freed), "freed": len(freed)}


def check(log, buf_meta, tasks, closed=True):
    """Raise InvariantError on the first violation; returns stats dict."""
    alloc_stats = check_allocations(log, closed)
    anc = []
    for i, rec in enumerate(log):
        if rec["iid"] != i:
            raise InvariantError("iid %d at position %d" % (rec["iid"], i))
        a = 0
        for d in rec["deps"]:
            if not 0 <= d < i:
                raise InvariantError("instruction %d depends on %d (not topological)" % (i, d))
            a |= anc[d] | (1 << d)
        anc.append(a)

    def is_anc(x, i):
        return x < 0 or (anc[i] >> x) & 1

    allocs = {}
    hosts = {}
    for bid, m in buf_meta.items():
        if m["host_init"] is not None:
            hosts[bid] = _A(m["extent"], None, host=True)
    ver = {bid: np.full(g.shape(m["extent"]), -3, dtype=np.int64) for bid, m in buf_meta.items()}
    for bid, m in buf_meta.items():
        if m["host_init"] is not None:
            ver[bid][...] = -1
    pending_ver = []
    cur_task = None
    nreads = 0

    def get(aid, bid, i):
        if aid == HOST_AID:
            return hosts[bid]
        if aid not in allocs:
            raise InvariantError("instruction %d uses unknown allocation %d" % (i, aid))
        A = allocs[aid]
        if A.freed is not None:
            raise InvariantError("instruction %d uses allocation %d after its free" % (i, aid))
        if A.alloc_iid is not None and not is_anc(A.alloc_iid, i):
            raise InvariantError("instruction %d uses allocation %d without a lifetime path" % (i, aid))
        return A

    def do_read(A, bx, i):
        sl = _sl(A.box, bx)
        ws = np.unique(A.writer[sl])
        for w in ws:
            if w >= 0 and not is_anc(int(w), i):
                raise InvariantError("RAW: instruction %d reads data of %d without a path" % (i, w))
        mask = np.zeros(A.writer.shape, dtype=bool)
        mask[sl] = True
        A.readers.append((i, mask))
        return A.token[sl]

    def do_write(A, bx, i, token):
        sl = _sl(A.box, bx)
        ws = np.unique(A.writer[sl])
        for w in ws:
            if w >= 0 and not is_anc(int(w), i):
                raise InvariantError("WAW: instruction %d overwrites %d without a path" % (i, w))
        mask = np.zeros(A.writer.shape, dtype=bool)
        mask[sl] = True
        keep = []
        for (r, rm) in A.readers:
            if r != i and (rm & mask).any() and not is_anc(r, i):
                raise InvariantError("WAR: instruction %d overwrites data read by %d without a path" % (i, r))
            rm2 = rm & ~mask
            if rm2.any():
                keep.append((r, rm2))
        A.readers = keep
        A.writer[sl] = i
        if token is not None:
            A.token[sl] = token

    def flush_ver():
        for bid, bx, k in pending_ver:
            ver[bid][_sl(buf_meta[bid]["extent"], bx)] = k
        pending_ver.clear()

    for i, rec in enumerate(log):
        kind = rec["kind"]
        if kind != "kernel" or rec["task"] != cur_task:
            flush_ver()
        cur_task = rec.get("task") if kind == "kernel" else None
        if kind == "alloc":
            allocs[rec["aid"]] = _A(_tobox(rec["box"]), i)
        elif kind == "free":
            A = get(rec["aid"], rec["buffer"], i)
            for r, _ in A.readers:
                if not is_anc(r, i):
                    raise InvariantError("free %d does not follow reader %d" % (i, r))
            for w in np.unique(A.writer):
                if w >= 0 and not is_anc(int(w), i):
                    raise InvariantError("free %d does not follow writer %d" % (i, w))
            A.freed = i
        elif kind == "copy":
            bid = rec["buffer"]
            S = get(rec["src_aid"], bid, i)
            for jb in rec["region"]:
                bx = _tobox(jb)
                if not g.box_contains(S.box, bx):
                    raise InvariantError("copy %d reads outside its source allocation" % i)
                tok = do_read(S, bx, i)
                if rec["dst_aid"] == USER_AID:
                    exp = ver[bid][_sl(buf_meta[bid]["extent"], bx)]
                    bad = (exp != -3) & (tok != exp)
                    if bad.any():
                        raise InvariantError("readback %d returns a stale value" % i)
                    nreads += int((exp != -3).sum())
                else:
                    D = get(rec["dst_aid"], bid, i)
                    if not g.box_contains(D.box, bx):
                        raise InvariantError("copy %d writes outside its destination allocation" % i)
                    do_write(D, bx, i, tok.copy())
        elif kind == "kernel":
            spec = tasks[rec["task"]]
            chunk = _tobox(rec["chunk"])
            reads, writes = {}, {}
            for (bid, mode, mp), aid in zip(spec["accesses"], rec["bindings"]):
                for bx in mapper_region(_norm_mapper(mp), chunk, buf_meta[bid]["extent"]):
                    if mode in READS:
                        reads.setdefault((bid, aid), []).append(bx)
                    if mode in WRITES:
                        writes.setdefault((bid, aid), []).append(bx)
            for (bid, aid), bxs in sorted(reads.items()):
                A = get(aid, bid, i)
                for bx in bxs:
                    if not g.box_contains(A.box, bx):
                        raise InvariantError("kernel %d reads outside its allocation" % i)
                    tok = do_read(A, bx, i)
                    exp = ver[bid][_sl(buf_meta[bid]["extent"], bx)]
                    bad = (exp != -3) & (tok != exp)
                    if bad.any():
                        raise InvariantError("kernel %d (task %d) reads a stale or missing value of buffer %d"
                                             % (i, rec["task"], bid))
                    nreads += int((exp != -3).sum())
            for (bid, aid), bxs in sorted(writes.items()):
                A = get(aid, bid, i)
                for bx in bxs:
                    if not g.box_contains(A.box, bx):
                        raise InvariantError("kernel %d writes outside its allocation" % i)
                    do_write(A, bx, i, i)
                    pending_ver.append((bid, bx, i))
        # horizons / epochs carry no data
    flush_ver()
    live = [aid for aid, A in allocs.items() if A.freed is None]
    return {"instructions": len(log), "checked_reads": nreads, "live_allocs": live, **alloc_stats}
