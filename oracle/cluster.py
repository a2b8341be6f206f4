"""Virtual-node mode: N nodes x D devices, each node with its own scheduler
(§2.4, §3.4, §4.2).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

P:L319-326 (§3.1): the task's kernel index space is split over the nodes
(command chunks), and each command chunk "a second time" over the node's local
devices.  P:L386-392 (§3.4): during command-graph generation every node
decides which buffer regions it must *push* to which peer and which regions it
must *await*; an await-push only knows the union of what it will receive.
Command-graph generation is replicated: every node runs the same
deterministic bookkeeping ("per-node replicated, deterministically
identical"), kept once here:

  owner[b]    RegionMap: node that last wrote each element (NONE: never
              written; ALL: host-initialised data, present on every node)
  holders[b]  RegionMap: bit set of nodes holding an up-to-date copy

R17 [readings]:
  * Node split: 1-D along dim 0 (R4 rule); the task's own split kind
    (1d / 2d) applies to the devices inside a node.
  * For a task, node m misses  reads_m(b) - {elements m holds}  (ignoring never
    written elements); each missing element is pushed by its owner.  Pushes
    are coalesced per (owner, receiver, buffer) into one push command
    (S:L278); the await-push region of m is the union.
  * Transfer id = (tid, buffer).
  * After the task: receivers hold what they received; a writer becomes the
    owner and the only holder of what it wrote; every other node marks it
    stale in its instruction-graph tracking.
  * Readback: node 0 gathers the box (owners push the parts it lacks); the
    result is node 0's user pointer.  Every node closes with an epoch.
"""

from . import geometry as g
from .program import CelError, READS, WRITES, mapper_region, split
from .scheduler import Runtime, _Cmd, _norm_mapper

NONE = -1
ALL = -2


class Cluster:
    """N virtual nodes of D devices each; API of oracle.scheduler.Runtime."""

    def __init__(self, n_nodes, devices_per_node, lookahead="auto", horizon_step=4, checks=True):
        assert n_nodes >= 1 and devices_per_node >= 1
        self.N = n_nodes
        self.D = devices_per_node
        self.nodes = [Runtime(devices_per_node, lookahead, horizon_step, checks) for _ in range(n_nodes)]
        for k, rt in enumerate(self.nodes):
            rt.node = k
        self.owner = {}
        self.holders = {}
        self.buf_meta = self.nodes[0].buf_meta
        self.readbacks = self.nodes[0].readbacks
        self.tasks = self.nodes[0].tasks
        self.shut = False

    @property
    def logs(self):
        return [rt.log for rt in self.nodes]

    def pilots(self):
        return [p for rt in self.nodes for p in rt.pilots]

    # ------------------------------------------------------------------ API
    def buffer_create(self, dims, extent, elem_size, host_init=None):
        bids = [rt.buffer_create(dims, extent, elem_size, host_init) for rt in self.nodes]
        bid = bids[0]
        ext = self.nodes[0].bufs[bid].extent
        self.owner[bid] = g.RegionMap(ext, ALL if host_init is not None else NONE)
        self.holders[bid] = g.RegionMap(ext, (1 << self.N) - 1 if host_init is not None else 0)
        return bid

    def _node_access(self, spec, chunk):
        """reads / writes {bid: Region} of one command chunk (R5 mappers)."""
        reads, writes = {}, {}
        if g.is_empty(chunk):
            return reads, writes
        for (bid, mode, mapper) in spec["accesses"]:
            reg = mapper_region(mapper, chunk, self.nodes[0].bufs[bid].extent)
            if not reg:
                continue
            if mode in READS:
                reads[bid] = g.region_union(reads.get(bid, ()), reg)
            if mode in WRITES:
                writes[bid] = g.region_union(writes.get(bid, ()), reg)
        return reads, writes

    def _transfers(self, need_by_node):
        """need_by_node: [{bid: Region}] per receiving node -> (pushes per node
        [(target, bid, Region)], awaits per node {bid: Region})."""
        pushes = [dict() for _ in range(self.N)]
        awaits = [dict() for _ in range(self.N)]
        for m in range(self.N):
            for b in sorted(need_by_node[m]):
                r = need_by_node[m][b]
                held = self.holders[b].region_where(lambda mask, m=m: (mask >> m) & 1)
                miss = g.region_difference(r, held)
                for piece, n in self.owner[b].query(miss):
                    if n < 0 or n == m:
                        continue
                    k = (m, b)
                    pushes[n][k] = g.region_union(pushes[n].get(k, ()), piece)
                    awaits[m][b] = g.region_union(awaits[m].get(b, ()), piece)
        plist = [[(m, b, reg) for (m, b), reg in sorted(p.items())] for p in pushes]
        return plist, awaits

    def task_submit(self, spec):
        if self.shut:
            raise CelError(CelError.STATE, "runtime shut down")
        user_spec = spec
        spec = dict(spec)
        spec["accesses"] = [(bid, mode, _norm_mapper(mp)) for (bid, mode, mp) in spec["accesses"]]
        for (bid, mode, mapper) in spec["accesses"]:
            if bid not in self.owner:
                raise CelError(CelError.INVALID, "no such buffer")
        rng = g.box(spec["range"][0], spec["range"][1])
        chunks = split(rng, self.N, "1d")
        acc = [self._node_access(spec, ch) for ch in chunks]
        # §4.4 overlapping writes across nodes
        for b in sorted({b for (_, w) in acc for b in w}):
            ws = [(n, acc[n][1][b]) for n in range(self.N) if b in acc[n][1]]
            for i in range(len(ws)):
                for j in range(i + 1, len(ws)):
                    if g.region_intersect(ws[i][1], ws[j][1]):
                        raise CelError(CelError.OVERLAPPING_WRITE,
                                       "nodes %d and %d write overlapping regions of buffer %d"
                                       % (ws[i][0], ws[j][0], b))
        reads, writes = {}, {}
        for (r, w) in acc:
            for b, x in r.items():
                reads[b] = g.region_union(reads.get(b, ()), x)
            for b, x in w.items():
                writes[b] = g.region_union(writes.get(b, ()), x)
        pushes, awaits = self._transfers([a[0] for a in acc])
        res = None
        for n, rt in enumerate(self.nodes):
            remote = {}
            for k in range(self.N):
                if k == n:
                    continue
                for b, x in acc[k][1].items():
                    remote[b] = g.region_union(remote.get(b, ()), x)
            r = rt.task_submit_node(user_spec, chunks[n], reads, writes, pushes[n], awaits[n], remote)
            res = r if res is None else res
        # replicated bookkeeping after the task
        for m in range(self.N):
            for b, reg in awaits[m].items():
                self.holders[b].apply(reg, lambda mask, m=m: mask | (1 << m))
        for n in range(self.N):
            for b, w in acc[n][1].items():
                self.owner[b].update(w, n)
                self.holders[b].update(w, 1 << n)
        return res

    def wait(self):
        for rt in self.nodes:
            rt.wait()

    def buffer_read(self, bid, rbox):
        if bid not in self.owner:
            raise CelError(CelError.INVALID, "no such buffer")
        rbox = g.box(rbox[0], rbox[1])
        rt0 = self.nodes[0]
        if not g.box_contains(rt0.bufs[bid].extent, rbox):
            raise CelError(CelError.OUT_OF_BOUNDS, "readback box outside extent")
        need = [dict() for _ in range(self.N)]
        need[0][bid] = (rbox,)
        pushes, awaits = self._transfers(need)
        rb = rt0.next_rb
        rt0.next_rb += 1
        rt0.readbacks[rb] = (bid, rbox)
        for n, rt in enumerate(self.nodes):
            c = _Cmd("epoch")
            if n == 0:
                c.readback = (rb, bid, rbox)
            c.pushes = pushes[n]
            c.awaits = awaits[n]
            rt._transfer_req(c)
            rt._epoch(c)
        for b, reg in awaits[0].items():
            self.holders[b].apply(reg, lambda mask: mask | 1)
        return rb

    def buffer_destroy(self, bid):
        for rt in self.nodes:
            rt.buffer_destroy(bid)
        del self.owner[bid], self.holders[bid]

    def shutdown(self):
        if self.shut:
            return
        for rt in self.nodes:
            rt.shutdown()
        self.shut = True
