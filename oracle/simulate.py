"""Byte simulator and sequential definition (test infrastructure; oracle).

simulate(): executes an instruction log in iid order — a topological order,
so sequential execution trivially satisfies every dependency (P:L518,
§4.1) — over per-allocation arrays (R15: an allocation is a dense row-major
array over its box; a copy moves exactly its region's bytes; a kernel
addresses its bound allocations at buffer coordinates).  Fresh allocations
are filled with a garbage pattern so a missing coherence copy shows up.

sequential(): the plain definition the instruction graph must reproduce
(semantic transparency): every task applied, in submission
order, to ONE global array per buffer over the whole kernel range — no
split, no allocations, no copies.
"""

import numpy as np

from . import geometry as g
from .kernels import Acc, run_kernel
from .program import apply_mapper
from .scheduler import HOST_AID, USER_AID, _norm_mapper

GARBAGE = np.uint32(0x7FC00BAD)      # a float32 NaN payload; never produced by a kernel


def _words(elem_size):
    assert elem_size % 4 == 0, "the simulator models 4-byte words"
    return elem_size // 4


def host_array(data, extent, elem_size):
    sh = g.shape(extent) + (_words(elem_size),)
    a = np.ascontiguousarray(data).reshape(-1).view(np.uint32)
    return a.reshape(sh).copy()


def _tobox(jb):
    return (tuple(jb[0]), tuple(jb[1]))


def _view(arr, abox, bx):
    b = abox[0]
    return arr[bx[0][0] - b[0]:bx[1][0] - b[0], bx[0][1] - b[1]:bx[1][1] - b[1],
               bx[0][2] - b[2]:bx[1][2] - b[2]]


class _NodeState:
    def __init__(self, rt, with_results):
        self.rt = rt
        self.meta = rt.buf_meta
        self.arrays = {}
        self.boxes = {}
        self.host = {}
        for bid, m in self.meta.items():
            if m["host_init"] is not None:
                self.host[bid] = host_array(m["host_init"], m["extent"], m["elem_size"])
        self.results = {}
        if with_results:
            for rb, (bid, rbox) in rt.readbacks.items():
                self.results[rb] = np.full(g.shape(rbox) + (_words(self.meta[bid]["elem_size"]),), GARBAGE,
                                           dtype=np.uint32)
        self.split = {}          # transfer -> dst aid of its split receive


def simulate(rt):
    """Run rt.log over arrays.  Returns {readback id: uint32 array}."""
    st = _NodeState(rt, True)
    for rec in rt.log:
        _step(st, rec)
    return st.results


def simulate_cluster(cl):
    """Virtual-node mode (oracle/cluster.py): run every node's log; a send
    publishes its box's bytes under (sender, message id); a receive / await
    receive takes the bytes of every pilot addressed to it (P:L534-544 receive
    arbitration: placement by the pilot's box) once they have been sent.  The
    nodes advance round-robin, each until it reaches a receive whose data is
    not yet sent.  Returns node 0's readbacks."""
    states = [_NodeState(rt, n == 0) for n, rt in enumerate(cl.nodes)]
    pilots = cl.pilots()
    sent = {}
    pcs = [0] * len(states)
    while True:
        progress = False
        for n, st in enumerate(states):
            log = st.rt.log
            while pcs[n] < len(log):
                rec = log[pcs[n]]
                if rec["kind"] in ("receive", "await_receive"):
                    tr = tuple(rec["transfer"])
                    reg = [_tobox(jb) for jb in rec["region"]]
                    mine = [p for p in pilots if p["receiver"] == n and tuple(p["transfer"]) == tr and
                            g.region_intersect((p["box"],), tuple(reg))]
                    if any((p["sender"], p["msg"]) not in sent for p in mine):
                        break
                    aid = rec["dst_aid"] if rec["kind"] == "receive" else st.split[tr]
                    for p in mine:
                        _view(st.arrays[aid], st.boxes[aid], p["box"])[...] = sent[(p["sender"], p["msg"])]
                elif rec["kind"] == "send":
                    bx = _tobox(rec["box"])
                    sent[(n, rec["msg"])] = _view(st.arrays[rec["src_aid"]], st.boxes[rec["src_aid"]], bx).copy()
                elif rec["kind"] == "split_receive":
                    st.split[tuple(rec["transfer"])] = rec["dst_aid"]
                else:
                    _step(st, rec)
                pcs[n] += 1
                progress = True
        if all(pcs[n] == len(st.rt.log) for n, st in enumerate(states)):
            return states[0].results
        if not progress:
            raise AssertionError("virtual-node simulation deadlocked at %s" % pcs)


def _step(st, rec):
    rt, meta, arrays, boxes, host, results = st.rt, st.meta, st.arrays, st.boxes, st.host, st.results
    if True:
        k = rec["kind"]
        if k == "alloc":
            bx = _tobox(rec["box"])
            words = _words(meta[rec["buffer"]]["elem_size"])
            arrays[rec["aid"]] = np.full(g.shape(bx) + (words,), GARBAGE, dtype=np.uint32)
            boxes[rec["aid"]] = bx
        elif k == "free":
            del arrays[rec["aid"]]
        elif k == "copy":
            bid = rec["buffer"]
            if rec["src_aid"] == HOST_AID:
                src, sbox = host[bid], meta[bid]["extent"]
            else:
                src, sbox = arrays[rec["src_aid"]], boxes[rec["src_aid"]]
            if rec["dst_aid"] == USER_AID:
                dst, dbox = results[rec["readback"]], rt.readbacks[rec["readback"]][1]
            else:
                dst, dbox = arrays[rec["dst_aid"]], boxes[rec["dst_aid"]]
            for jb in rec["region"]:
                bx = _tobox(jb)
                _view(dst, dbox, bx)[...] = _view(src, sbox, bx)
        elif k == "kernel":
            spec = rt.tasks[rec["task"]]
            chunk = _tobox(rec["chunk"])
            bxs, accs = [], []
            for (bid, mode, mapper), aid in zip(spec["accesses"], rec["bindings"]):
                ext = meta[bid]["extent"]
                bxs.append(apply_mapper(mapper, chunk, ext))
                accs.append(Acc(arrays[aid], boxes[aid], ext) if aid > 0 else None)
            run_kernel(spec, bxs, accs)


def sequential(program):
    """Apply the program's tasks in order to one global array per buffer.
    Returns ({readback index: uint32 array}, {readback index: bool mask of
    defined elements})."""
    bufs, defined, meta = [], [], []
    for b in program["buffers"]:
        ext = g.box([0] * b["dims"], list(b["extent"]))
        words = _words(b["elem_size"])
        meta.append(ext)
        if b.get("host_init") is not None:
            bufs.append(host_array(b["host_init"], ext, b["elem_size"]))
            defined.append(np.ones(g.shape(ext), dtype=bool))
        else:
            bufs.append(np.full(g.shape(ext) + (words,), GARBAGE, dtype=np.uint32))
            defined.append(np.zeros(g.shape(ext), dtype=bool))
    results, masks = {}, {}
    rb = 0
    for op in program["ops"]:
        if op[0] == "task":
            spec = dict(op[1])
            spec["accesses"] = [(bid, mode, _norm_mapper(mp)) for (bid, mode, mp) in spec["accesses"]]
            rng = g.box(spec["range"][0], spec["range"][1])
            if g.is_empty(rng):
                continue
            bxs, accs = [], []
            ok = True
            for (bid, mode, mapper) in spec["accesses"]:
                bx = apply_mapper(mapper, rng, meta[bid])
                bxs.append(bx)
                accs.append(Acc(bufs[bid], meta[bid], meta[bid]))
                if mode in ("read", "read_write") and not g.is_empty(bx):
                    ok = ok and bool(_view(defined[bid], meta[bid], bx).all())
            run_kernel(spec, bxs, accs)
            for (bid, mode, mapper), bx in zip(spec["accesses"], bxs):
                if mode in ("write", "read_write") and not g.is_empty(bx):
                    _view(defined[bid], meta[bid], bx)[...] = ok
        elif op[0] == "read":
            bid, rbox = op[1], g.box(op[2][0], op[2][1])
            results[rb] = _view(bufs[bid], meta[bid], rbox).copy()
            masks[rb] = _view(defined[bid], meta[bid], rbox).copy()
            rb += 1
    return results, masks
