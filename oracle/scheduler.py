"""Oracle scheduler: task tracking, horizons, lookahead and IDAG generation.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Follows PAPER.md §2.4,
§3 and §4.3 step by step, in the order and notation of the paper; where the
paper is silent the DESIGN.md reading (R0-R17) is cited.

Topology (R0, §3.2): one node, G devices D0..D(G-1); memory ids
M0 = user host, M1 = pinned host (never used: B200/NVSwitch supports d2d,
so host staging P:L380 is never emitted), M(2+d) = device d.

Instruction log record (one dict per instruction, iid order):
  alloc   {iid, kind, task, buffer, aid, mem, box, deps}
  free    {iid, kind, task, buffer, aid, mem, deps}
  copy    {iid, kind, task, buffer, reason, src_aid, src_mem, dst_aid, dst_mem, region, deps}
          reason in {resize, coherence, readback}; aid -1 = the buffer's implicit
          M0 host allocation (R6), aid -2 = the user pointer of a readback (R13)
  kernel  {iid, kind, task, device, chunk, bindings, deps}
  horizon {iid, kind, task, deps}
  epoch   {iid, kind, task, deps}
Virtual-node mode (oracle/cluster.py) adds, per node:
  send          {iid, kind, task, buffer, target, msg, src_aid, src_mem, box, deps}
  receive       {iid, kind, task, buffer, transfer, dst_aid, dst_mem, region, deps}
  split_receive {iid, kind, task, buffer, transfer, dst_aid, dst_mem, region, deps}
  await_receive {iid, kind, task, buffer, transfer, region, deps}
  transfer = [tid, buffer] (S:L261 convention); src/dst of sends and receives
  is the node's M1 staging allocation ("coherence copy to host memory").
Boxes are [[min0,min1,min2],[max0,max1,max2]]; regions are lists of boxes in
R2 canonical order.
"""

from . import geometry as g
from .program import CelError, READS, WRITES, apply_mapper, mapper_region, split

NONE = -1          # "no writer" (uninitialised) in writer maps
HOST_AID = -1      # implicit M0 allocation of a host-initialised buffer (R6)
USER_AID = -2      # user destination pointer of a readback (R13)


def _jbox(b):
    return [list(b[0]), list(b[1])]


def _jregion(r):
    return [_jbox(b) for b in r]


class _Alloc:
    __slots__ = ("aid", "buffer", "mem", "box", "iid", "last_writer", "readers")

    def __init__(self, aid, buffer, mem, box, iid, init_writer):
        self.aid = aid
        self.buffer = buffer
        self.mem = mem
        self.box = box
        self.iid = iid                       # alloc instruction (None for HOST_AID)
        # R12: per-allocation last writer / readers-since-last-write
        self.last_writer = g.RegionMap(box, init_writer)
        self.readers = g.RegionMap(box, frozenset())


class _Buf:
    def __init__(self, bid, dims, extent, elem_size, host_init, fallback_iid):
        self.bid = bid
        self.dims = dims
        self.extent = extent
        self.elem_size = elem_size
        self.host_init = host_init
        # P:L372 §3.3: "which instruction has been its local original producer"
        self.orig_writer = g.RegionMap(extent, fallback_iid if host_init else NONE)
        # "which buffer subregions are locally up-to-date on what memory ids"
        self.uptodate = g.RegionMap(extent, 1 if host_init else 0)   # bit m = memory Mm
        self.live = {}                       # mem -> [ _Alloc ]  (non-overlapping)
        self.host = (_Alloc(HOST_AID, bid, 0, extent, None, fallback_iid) if host_init else None)


class TaskGraph:
    """§2.4 task graph, reduced to what the IDAG path consumes: element-granular
    dependencies -> critical-path length -> horizon placement
    (R7 [reading]: step 4, critical-path trigger only)."""

    def __init__(self, step):
        self.step = step
        self.next_tid = 1
        self.cp = {0: 0}                     # tid 0 = init epoch
        self.fallback = 0
        self.pending_h = None
        self.max_cp = 0
        self.cp_ref = 0
        self.last_writer = {}
        self.readers = {}
        self.initialized = {}

    def add_buffer(self, bid, extent, host_init):
        self.last_writer[bid] = g.RegionMap(extent, self.fallback if host_init else NONE)
        self.readers[bid] = g.RegionMap(extent, frozenset())
        self.initialized[bid] = (extent,) if host_init else ()

    def drop_buffer(self, bid):
        del self.last_writer[bid], self.readers[bid], self.initialized[bid]

    def _new(self):
        t = self.next_tid
        self.next_tid += 1
        return t

    def submit(self, reads, writes):
        """reads/writes: {bid: Region}.  Returns tid.  RAW/WAR/WAW at element
        granularity; fallback edge to epoch/applied horizon."""
        deps = set()
        for b, r in reads.items():
            deps |= {v for _, v in self.last_writer[b].query(r) if v >= 0}
        for b, w in writes.items():
            for _, s in self.readers[b].query(w):
                deps |= s
            deps |= {v for _, v in self.last_writer[b].query(w) if v >= 0}
        if not deps:
            deps = {self.fallback}
        tid = self._new()
        self.cp[tid] = 1 + max(self.cp[d] for d in deps)
        for b, r in reads.items():
            self.readers[b].apply(r, lambda s, t=tid: s | {t})
        for b, w in writes.items():
            self.last_writer[b].update(w, tid)
            self.readers[b].update(w, frozenset())
            self.initialized[b] = g.region_union(self.initialized[b], w)
        self.max_cp = max(self.max_cp, self.cp[tid])
        return tid

    def horizon_due(self):
        return self.max_cp - self.cp_ref >= self.step

    def _subsume(self, h):
        for b in self.last_writer:
            self.last_writer[b].map_values(lambda v: h if 0 <= v < h else v)
            self.readers[b].map_values(lambda s: frozenset(h if x < h else x for x in s))

    def horizon(self):
        """a horizon bounds tracking; applying the previous
        one subsumes older tracker entries (R7)."""
        tid = self._new()
        self.cp[tid] = self.max_cp
        self.cp_ref = self.max_cp
        if self.pending_h is not None:
            self._subsume(self.pending_h)
            self.fallback = self.pending_h
        self.pending_h = tid
        return tid

    def epoch(self):
        tid = self._new()
        self.cp[tid] = 0
        self._subsume(tid)
        self.fallback = tid
        self.pending_h = None
        self.max_cp = 0
        self.cp_ref = 0
        return tid


class _Cmd:
    """A command of the (single-node) command graph: one execution command per
    task, or a horizon / epoch / destroy."""

    def __init__(self, kind, tid=None):
        self.kind = kind
        self.tid = tid
        self.spec = None
        self.chunks = []
        self.reads = {}       # (d, bid) -> Region
        self.writes = {}      # (d, bid) -> Region
        self.req = {}         # (d, bid) -> Box   (R9: bbox of reads ∪ writes)
        self.readback = None  # (rb_id, bid, box)
        self.destroy = []     # bids
        self.shutdown = False
        # virtual-node mode (oracle/cluster.py): this node's transfers for the task
        self.pushes = []      # [(target node, bid, Region)] sorted by (target, bid)
        self.awaits = {}      # bid -> Region awaited from other nodes
        self.remote_writes = {}   # bid -> Region written by other nodes in this task


class Runtime:
    """Oracle counterpart of the C-ABI runtime (include/cel.h), no GPU."""

    def __init__(self, n_devices, lookahead="auto", horizon_step=4, checks=True):
        assert n_devices >= 1
        assert lookahead in ("none", "auto", "infinite")
        self.G = n_devices
        self.mode = lookahead
        self.checks = checks
        self.tdag = TaskGraph(horizon_step)
        self.bufs = {}
        self.buf_meta = {}
        self.tasks = {}
        self.readbacks = {}
        self.warnings = []
        self.log = []
        self.next_bid = 0
        self.next_aid = 1
        self.next_rb = 0
        self.allocs = {}                     # aid -> _Alloc (live)
        self.alloc_iid = {}
        self.front = set()
        self.fallback = 0
        self.pending_h = None
        self.queue = []
        self.counter = 0
        self.flushes = 0
        self.shut = False
        self.node = 0                        # node id in virtual-node mode
        self.next_msg = 0                    # P:L400 "locally unique message id"
        self.pilots = []                     # P:L401 pilot messages of this node's sends
        # init epoch, iid 0 / tid 0 (P:L238 epochs; "the first task is an epoch")
        self.log.append({"iid": 0, "kind": "epoch", "task": 0, "deps": []})
        self.front = {0}

    # ------------------------------------------------------------------ API
    def buffer_create(self, dims, extent, elem_size, host_init=None):
        if self.shut:
            raise CelError(CelError.STATE, "runtime shut down")
        if not 1 <= dims <= 3 or len(extent) != dims or any(e <= 0 for e in extent) or elem_size <= 0:
            raise CelError(CelError.INVALID, "bad buffer")
        bid = self.next_bid
        self.next_bid += 1
        ext = g.box([0] * dims, list(extent))
        self.bufs[bid] = _Buf(bid, dims, ext, elem_size, host_init is not None, self.fallback)
        self.buf_meta[bid] = {"dims": dims, "extent": ext, "elem_size": elem_size,
                              "host_init": host_init}
        self.tdag.add_buffer(bid, ext, host_init is not None)
        return bid

    def task_submit(self, spec):
        """Returns (tid, status): status 1 = uninitialised-read warning."""
        if self.shut:
            raise CelError(CelError.STATE, "runtime shut down")
        cmd = self._prepare(spec)          # validation + split + mappers + checks
        reads, writes = {}, {}
        for (d, b), r in cmd.reads.items():
            reads[b] = g.region_union(reads.get(b, ()), r)
        for (d, b), w in cmd.writes.items():
            writes[b] = g.region_union(writes.get(b, ()), w)
        return self._submit(cmd, reads, writes)

    def task_submit_node(self, spec, node_range, reads, writes, pushes, awaits, remote_writes):
        """Virtual-node mode: this node's share of a
        task -- its command chunk `node_range` split "a second time" over the
        local devices -- plus the push / await-push transfers the replicated
        command-graph generation derived for it (oracle/cluster.py).  The task
        graph sees the whole task (`reads` / `writes` over all nodes)."""
        if self.shut:
            raise CelError(CelError.STATE, "runtime shut down")
        cmd = self._prepare(spec, node_range)
        cmd.pushes = list(pushes)
        cmd.awaits = dict(awaits)
        cmd.remote_writes = dict(remote_writes)
        self._transfer_req(cmd)
        return self._submit(cmd, reads, writes)

    def _submit(self, cmd, reads, writes):
        status = 0
        if self.checks:
            for bid in sorted(reads):
                un = g.region_difference(reads[bid], self.tdag.initialized[bid])
                if un:
                    status = 1
                    self.warnings.append(("uninitialized_read", bid, un))
        tid = self.tdag.submit(reads, writes)
        cmd.tid = tid
        self.tasks[tid] = cmd.spec
        self._push(cmd)
        if self.tdag.horizon_due():
            h = _Cmd("horizon", self.tdag.horizon())
            self._push(h)
        return tid, status

    def _transfer_req(self, cmd):
        """P:L398 / P:L417: pushed data is staged in, and awaited data received
        into, one contiguous M1 allocation per buffer (requirement key d = -1,
        memory 2 + d = M1), covering every transferred region of the command."""
        boxes = {}
        for (_, b, reg) in cmd.pushes:
            boxes.setdefault(b, []).extend(reg)
        for b, reg in cmd.awaits.items():
            boxes.setdefault(b, []).extend(reg)
        for b, bs in boxes.items():
            cmd.req[(-1, b)] = g.bounding_box(bs)

    def wait(self):
        self._epoch(_Cmd("epoch"))

    def buffer_read(self, bid, rbox):
        if bid not in self.bufs:
            raise CelError(CelError.INVALID, "no such buffer")
        rbox = g.box(rbox[0], rbox[1])
        if not g.box_contains(self.bufs[bid].extent, rbox):
            raise CelError(CelError.OUT_OF_BOUNDS, "readback box outside extent")
        rb = self.next_rb
        self.next_rb += 1
        self.readbacks[rb] = (bid, rbox)
        c = _Cmd("epoch")
        c.readback = (rb, bid, rbox)
        self._epoch(c)
        return rb

    def buffer_destroy(self, bid):
        if bid not in self.bufs:
            raise CelError(CelError.INVALID, "no such buffer")
        self._flush()
        c = _Cmd("destroy")
        c.destroy = [bid]
        self._compile(c, {})
        self.tdag.drop_buffer(bid)

    def shutdown(self):
        if self.shut:
            return
        self._flush()
        if self.bufs:
            c = _Cmd("destroy")
            c.destroy = sorted(self.bufs)
            self._compile(c, {})
            for bid in c.destroy:
                self.tdag.drop_buffer(bid)
        self._epoch(_Cmd("epoch"))
        self.shut = True

    # ------------------------------------------------------------ prepare
    def _prepare(self, spec, node_range=None):
        dims = spec["dims"]
        if not 1 <= dims <= 3:
            raise CelError(CelError.INVALID, "bad dims")
        rng = g.box(spec["range"][0], spec["range"][1]) if node_range is None else node_range
        spec = dict(spec)
        spec["accesses"] = [(bid, mode, _norm_mapper(mp)) for (bid, mode, mp) in spec["accesses"]]
        for (bid, mode, mapper) in spec["accesses"]:
            if bid not in self.bufs:
                raise CelError(CelError.INVALID, "no such buffer")
            if mode not in ("read", "write", "read_write"):
                raise CelError(CelError.INVALID, "bad mode")
        cmd = _Cmd("task")
        cmd.spec = spec
        cmd.chunks = split(rng, self.G, spec.get("split", "1d"))
        for d, ch in enumerate(cmd.chunks):
            if g.is_empty(ch):
                continue
            for (bid, mode, mapper) in spec["accesses"]:
                reg = mapper_region(mapper, ch, self.bufs[bid].extent)
                if not reg:
                    continue
                if mode in READS:
                    cmd.reads[(d, bid)] = g.region_union(cmd.reads.get((d, bid), ()), reg)
                if mode in WRITES:
                    cmd.writes[(d, bid)] = g.region_union(cmd.writes.get((d, bid), ()), reg)
        # §4.4 Overlapping-write detection: error, state unchanged
        for bid in sorted({b for (_, b) in cmd.writes}):
            ws = [(d, cmd.writes[(d, bid)]) for d in range(self.G) if (d, bid) in cmd.writes]
            for i in range(len(ws)):
                for j in range(i + 1, len(ws)):
                    if g.region_intersect(ws[i][1], ws[j][1]):
                        raise CelError(CelError.OVERLAPPING_WRITE,
                                       "devices %d and %d write overlapping regions of buffer %d"
                                       % (ws[i][0], ws[j][0], bid))
        for key in set(cmd.reads) | set(cmd.writes):
            cmd.req[key] = g.bounding_box(list(cmd.reads.get(key, ())) + list(cmd.writes.get(key, ())))
        return cmd

    # ----------------------------------------------------------- lookahead
    def _anticipated(self, cmds):
        """bbox of all requirements observed while queued, per (buffer, memory)."""
        ant = {}
        for c in cmds:
            for (d, b), bx in c.req.items():
                k = (b, 2 + d)
                ant[k] = g.bounding_box([ant.get(k, g.EMPTY), bx])
        return ant

    def _is_allocating(self, cmd):
        """would compiling it emit an alloc?  R8 [reading]: test req
        containment against live allocations and the queued requirements."""
        ant = self._anticipated(self.queue) if self.queue else {}
        for (d, b), bx in sorted(cmd.req.items()):
            m = 2 + d
            if any(g.box_contains(a.box, bx) for a in self.bufs[b].live.get(m, [])):
                continue
            if (b, m) in ant and g.box_contains(ant[(b, m)], bx):
                continue
            return True
        return False

    def _push(self, cmd):
        """§4.3 Command Queueing + Lookahead Heuristic."""
        if self.mode == "none":
            self._compile(cmd, {})
            return
        if cmd.kind == "horizon":
            if not self.queue:
                self._compile(cmd, {})
                return
            self.queue.append(cmd)
            self.counter += 1
            if self.mode == "auto" and self.counter >= 2:   # P:L584 "two horizons"
                self._flush()
            return
        alloc = self._is_allocating(cmd)
        if self.mode == "auto" and not self.queue and not alloc:
            self._compile(cmd, {})
            return
        self.queue.append(cmd)
        if alloc:
            self.counter = 0

    def _flush(self):
        if not self.queue:
            return
        q = self.queue
        ant = self._anticipated(q)
        self.queue = []
        self.counter = 0
        self.flushes += 1
        for c in q:
            self._compile(c, ant)

    def _epoch(self, cmd):
        self._flush()
        cmd.tid = self.tdag.epoch()
        self._compile(cmd, {})

    # ---------------------------------------------------------- emission
    def _emit(self, rec, deps):
        iid = len(self.log)
        deps = set(deps)
        deps.discard(None)
        if not deps:
            deps = {self.fallback}        # R12: fallback to last epoch / applied horizon
        rec = dict(rec)
        rec["iid"] = iid
        rec["deps"] = sorted(deps)
        self.front -= deps
        self.front.add(iid)
        self.log.append(rec)
        return iid

    def _alloc(self, bid, mem, bx, tid):
        aid = self.next_aid
        self.next_aid += 1
        iid = self._emit({"kind": "alloc", "task": tid, "buffer": bid, "aid": aid, "mem": mem,
                          "box": _jbox(bx)}, [])
        a = _Alloc(aid, bid, mem, bx, iid, NONE)
        self.allocs[aid] = a
        self.alloc_iid[aid] = iid
        self.bufs[bid].live.setdefault(mem, []).append(a)
        return a

    def _free(self, a, tid):
        deps = {a.iid}
        deps |= {v for v in a.last_writer.values() if v >= 0}
        for s in a.readers.values():
            deps |= s
        self._emit({"kind": "free", "task": tid, "buffer": a.buffer, "aid": a.aid, "mem": a.mem}, deps)
        self.bufs[a.buffer].live[a.mem].remove(a)
        del self.allocs[a.aid]

    def _copy(self, tid, bid, reason, src, dst, reg, dst_aid=None, dst_mem=None):
        """Table 1 `copy` with R12 deps: dataflow on the source
        allocation's last writers, anti/output on the destination's."""
        deps = set()
        if src.iid is not None:
            deps.add(src.iid)
        for _, v in src.last_writer.query(reg):
            if v >= 0:
                deps.add(v)
        if dst is not None:
            deps.add(dst.iid)
            for _, s in dst.readers.query(reg):
                deps |= s
            for _, v in dst.last_writer.query(reg):
                if v >= 0:
                    deps.add(v)
        iid = self._emit({"kind": "copy", "task": tid, "buffer": bid, "reason": reason,
                          "src_aid": src.aid, "src_mem": src.mem,
                          "dst_aid": dst.aid if dst is not None else dst_aid,
                          "dst_mem": dst.mem if dst is not None else dst_mem,
                          "region": _jregion(reg)}, deps)
        src.readers.apply(reg, lambda s: s | {iid})
        if dst is not None:
            dst.last_writer.update(reg, iid)
            dst.readers.update(reg, frozenset())
        return iid

    @staticmethod
    def _pick_source(mask, m_dst):
        """R10 [reading]: lowest device memory != destination holding the
        element, else M1, else M0."""
        m = 2
        while (mask >> m) != 0:
            if (mask >> m) & 1 and m != m_dst:
                return m
            m += 1
        if mask & 2:
            return 1
        if mask & 1:
            return 0
        return None

    def _source_parts(self, buf, need, m_dst):
        """Producer split: partition `need` by (original producer
        p, source memory s, source allocation) -> {(p, s, aid): Region}."""
        parts = {}
        for reg, mask in buf.uptodate.query(need):
            s = self._pick_source(mask, m_dst)
            if s is None:
                continue
            srcs = [buf.host] if s == 0 else sorted(buf.live.get(s, []), key=lambda a: a.aid)
            for a in srcs:
                part = g.region_intersect(reg, (a.box,))
                if not part:
                    continue
                for r2, p in buf.orig_writer.query(part):
                    k = (p, s, a.aid)
                    parts[k] = g.region_union(parts.get(k, ()), r2)
        return parts

    def _compile(self, cmd, ant):
        if cmd.kind == "task":
            self._compile_task(cmd, ant)
        elif cmd.kind == "horizon":
            self._compile_horizon(cmd)
        elif cmd.kind == "epoch":
            self._compile_epoch(cmd)
        elif cmd.kind == "destroy":
            for bid in cmd.destroy:            # R14 / P:L365-366
                buf = self.bufs[bid]
                for a in sorted([a for lst in buf.live.values() for a in lst], key=lambda a: a.aid):
                    self._free(a, None)
                del self.bufs[bid]

    def _allocate(self, cmd, ant):
        """R9 allocation (Fig. 3; resize chain alloc -> copy -> free)
        for every requirement of the command, M1 (d = -1) first.  Returns the
        binding (d, bid) -> allocation."""
        tid = cmd.tid
        keys = sorted(cmd.req, key=lambda k: (k[0], k[1]))     # device asc, buffer asc
        binding = {}
        for (d, b) in keys:
            req = cmd.req[(d, b)]
            m = 2 + d
            buf = self.bufs[b]
            live = buf.live.get(m, [])
            hit = [a for a in live if g.box_contains(a.box, req)]
            if hit:
                binding[(d, b)] = hit[0]
                continue
            bx = g.bounding_box([req, ant.get((b, m), g.EMPTY)])       # P:L589 widening
            while True:
                merged = [a for a in live if not g.is_empty(g.box_intersect(a.box, bx))]
                nb = g.bounding_box([bx] + [a.box for a in merged])
                if nb == bx:
                    break
                bx = nb
            new = self._alloc(b, m, bx, tid)
            utd = buf.uptodate.region_where(lambda mask, m=m: (mask >> m) & 1)
            for a in sorted(merged, key=lambda a: a.aid):
                src_reg = g.region_intersect((a.box,), utd)
                for reg, p in buf.orig_writer.query(src_reg):
                    self._copy(tid, b, "resize", a, new, reg)
                self._free(a, tid)
            binding[(d, b)] = new
        return binding

    def _transfers(self, cmd, binding, readback_consumer=False):
        """Virtual-node mode, §3.4 Peer-to-Peer Communication.
        Outbound: the pushed region is made coherent in M1 ("a
        coherence copy to host memory"), then one send per rectangle of each
        original-producer fragment ("again subject to producer split"), each
        with a locally unique message id and a pilot for the receiver.
        Inbound: if every consumer reads the same part of the
        awaited region (or there is one consumer) one receive into M1;
        otherwise a split receive followed by one await receive per
        consumer-split fragment (R17 [reading]: the fragments are the atoms of
        the consumers' regions, refined device by device in ascending order)."""
        tid = cmd.tid
        for (target, b, reg) in cmd.pushes:
            buf = self.bufs[b]
            m1 = binding[(-1, b)]
            need = g.region_difference(reg, buf.uptodate.region_where(lambda mask: (mask >> 1) & 1))
            need = g.region_intersect(need, buf.uptodate.region_where(lambda mask: mask != 0))
            if need:
                parts = self._source_parts(buf, need, 1)
                for (p, s_, aid) in sorted(parts):
                    src = buf.host if aid == HOST_AID else self.allocs[aid]
                    self._copy(tid, b, "coherence", src, m1, parts[(p, s_, aid)])
                for k in sorted(parts):
                    buf.uptodate.apply(parts[k], lambda mask: mask | 2)
            for reg2, p in buf.orig_writer.query(reg):
                for bx in reg2:
                    deps = {m1.iid}
                    deps |= {v for _, v in m1.last_writer.query((bx,)) if v >= 0}
                    msg = self.next_msg
                    self.next_msg += 1
                    iid = self._emit({"kind": "send", "task": tid, "buffer": b, "target": target, "msg": msg,
                                      "src_aid": m1.aid, "src_mem": 1, "box": _jbox(bx)}, deps)
                    m1.readers.apply((bx,), lambda s, iid=iid: s | {iid})
                    self.pilots.append({"sender": self.node, "msg": msg, "receiver": target,
                                        "transfer": (tid, b), "box": bx})
        for b in sorted(cmd.awaits):
            reg = cmd.awaits[b]
            buf = self.bufs[b]
            m1 = binding[(-1, b)]
            if readback_consumer:
                consumers = [reg]
            else:
                consumers = []
                for d in range(self.G):
                    c = g.region_intersect(cmd.reads.get((d, b), ()), reg)
                    if c:
                        consumers.append(c)
            deps = {m1.iid}
            for _, s_ in m1.readers.query(reg):
                deps |= s_
            deps |= {v for _, v in m1.last_writer.query(reg) if v >= 0}
            rec = {"task": tid, "buffer": b, "transfer": [tid, b], "dst_aid": m1.aid, "dst_mem": 1,
                   "region": _jregion(reg)}
            if len(set(consumers)) <= 1:
                iid = self._emit(dict(rec, kind="receive"), deps)
                frags = [(reg, iid)]
            else:
                sr = self._emit(dict(rec, kind="split_receive"), deps)
                atoms = [reg]
                for c in consumers:
                    nxt = []
                    for a in atoms:
                        i = g.region_intersect(a, c)
                        o = g.region_difference(a, c)
                        if i:
                            nxt.append(i)
                        if o:
                            nxt.append(o)
                    atoms = nxt
                frags = []
                for a in atoms:
                    frags.append((a, self._emit({"kind": "await_receive", "task": tid, "buffer": b,
                                                 "transfer": [tid, b], "region": _jregion(a)}, {sr})))
            for r, iid in frags:
                m1.last_writer.update(r, iid)
                m1.readers.update(r, frozenset())
                buf.orig_writer.update(r, iid)
            buf.uptodate.update(reg, 2)

    def _compile_task(self, cmd, ant):
        tid = cmd.tid
        G = self.G
        binding = self._allocate(cmd, ant)
        keys = sorted(k for k in cmd.req if k[0] >= 0)          # device asc, buffer asc
        if cmd.pushes or cmd.awaits:
            self._transfers(cmd, binding)
        # R10 coherence copies, masks as they stood before this task
        updates = []
        for (d, b) in keys:
            r = cmd.reads.get((d, b), ())
            if not r:
                continue
            m = 2 + d
            buf = self.bufs[b]
            need = g.region_difference(r, buf.uptodate.region_where(lambda mask, m=m: (mask >> m) & 1))
            need = g.region_intersect(need, buf.uptodate.region_where(lambda mask: mask != 0))
            if not need:
                continue
            parts = self._source_parts(buf, need, m)
            for (p, s, aid) in sorted(parts):
                src = buf.host if aid == HOST_AID else self.allocs[aid]
                self._copy(tid, b, "coherence", src, binding[(d, b)], parts[(p, s, aid)])
                updates.append((b, parts[(p, s, aid)], m))
        for (b, reg, m) in updates:
            self.bufs[b].uptodate.apply(reg, lambda mask, m=m: mask | (1 << m))
        # R11 device kernels ("one device kernel instruction per device")
        kernels = {}
        for d in range(G):
            ch = cmd.chunks[d]
            if g.is_empty(ch):
                continue
            deps = set()
            bufs_d = sorted({b for (dd, b) in keys if dd == d})
            for b in bufs_d:
                a = binding[(d, b)]
                deps.add(a.iid)
                for _, v in a.last_writer.query(cmd.reads.get((d, b), ())):
                    if v >= 0:
                        deps.add(v)
                w = cmd.writes.get((d, b), ())
                for _, s in a.readers.query(w):
                    deps |= s
                for _, v in a.last_writer.query(w):
                    if v >= 0:
                        deps.add(v)
            bindings = []
            for (bid, mode, mapper) in cmd.spec["accesses"]:
                a = binding.get((d, bid))
                bindings.append(a.aid if a is not None else 0)
            k = self._emit({"kind": "kernel", "task": tid, "device": d, "chunk": _jbox(ch),
                            "bindings": bindings}, deps)
            for b in bufs_d:
                a = binding[(d, b)]
                r = cmd.reads.get((d, b), ())
                if r:
                    a.readers.apply(r, lambda s, k=k: s | {k})
                w = cmd.writes.get((d, b), ())
                if w:
                    a.last_writer.update(w, k)
                    a.readers.update(w, frozenset())
            kernels[d] = k
        for (d, b) in keys:
            w = cmd.writes.get((d, b), ())
            if w:
                self.bufs[b].orig_writer.update(w, kernels[d])
                self.bufs[b].uptodate.update(w, 1 << (2 + d))
        # virtual-node mode: what other nodes wrote in this task is stale here
        for b in sorted(cmd.remote_writes):
            r = cmd.remote_writes[b]
            self.bufs[b].uptodate.update(r, 0)
            self.bufs[b].orig_writer.update(r, NONE)

    def _subsume(self, h):
        """Horizon/epoch application ("limiting the set of ...
        original producers"; R7): values older than h are replaced by h."""
        f = lambda v: h if 0 <= v < h else v
        fs = lambda s: frozenset(h if x < h else x for x in s)
        for buf in self.bufs.values():
            buf.orig_writer.map_values(f)
            allocs = [a for lst in buf.live.values() for a in lst]
            if buf.host is not None:
                allocs.append(buf.host)
            for a in allocs:
                a.last_writer.map_values(f)
                a.readers.map_values(fs)

    def _compile_horizon(self, cmd):
        # a horizon "depends on all instructions on the current execution front"
        h = self._emit({"kind": "horizon", "task": cmd.tid}, set(self.front))
        if self.pending_h is not None:
            self._subsume(self.pending_h)
            self.fallback = self.pending_h
        self.pending_h = h

    def _compile_epoch(self, cmd):
        if cmd.pushes or cmd.awaits:          # virtual-node readback gather (oracle/cluster.py)
            binding = self._allocate(cmd, {})
            self._transfers(cmd, binding, readback_consumer=True)
        if cmd.readback is not None:
            rb, bid, rbox = cmd.readback
            buf = self.bufs[bid]
            need = g.region_intersect((rbox,), buf.uptodate.region_where(lambda mask: mask != 0))
            parts = self._source_parts(buf, need, 0) if need else {}
            for (p, s, aid) in sorted(parts):
                src = buf.host if aid == HOST_AID else self.allocs[aid]
                iid = self._copy(cmd.tid, bid, "readback", src, None, parts[(p, s, aid)],
                                 dst_aid=USER_AID, dst_mem=0)
                self.log[iid]["readback"] = rb
        e = self._emit({"kind": "epoch", "task": cmd.tid}, set(self.front))
        self._subsume(e)
        self.fallback = e
        self.pending_h = None


# ---------------------------------------------------------------- helpers
def _norm_mapper(mp):
    kind = mp[0]
    if kind == "fixed":
        return ("fixed", g.box(mp[1][0], mp[1][1]))
    if kind == "remap":
        kd = tuple(mp[2]) + (-1,) * (3 - len(mp[2]))
        mn = tuple(mp[1][0]) + (0,) * (3 - len(mp[1][0]))
        mx = tuple(mp[1][1]) + (1,) * (3 - len(mp[1][1]))
        return ("remap", (mn, mx), kd)
    if kind in ("neighborhood", "neighborhood_axes"):
        return (kind, tuple(mp[1]) + (0,) * (3 - len(mp[1])))
    return (kind,)


def counts(log):
    """Instruction counts by kind (copies by reason and memory pair)."""
    c = {}
    for r in log:
        k = r["kind"]
        if k == "copy":
            if r["reason"] == "coherence":
                if r["src_mem"] >= 2 and r["dst_mem"] >= 2:
                    k = "copy_d2d"
                elif r["src_mem"] == 0:
                    k = "copy_h2d"
                else:
                    k = "copy_other"
            else:
                k = "copy_" + r["reason"]
        c[k] = c.get(k, 0) + 1
    return c
