"""Pins for oracle/scheduler.py: the paper's worked example (Fig. 4), the
lookahead claims of §4.3, horizon placement, diagnostics, and semantic
transparency against the plain sequential definition on random programs."""

import json
import os

import numpy as np
import pytest

from oracle import geometry as g
from oracle.invariants import InvariantError, check
from oracle.program import CelError
from oracle.scheduler import Runtime, counts
from workloads.driver import run_program
from oracle.simulate import sequential, simulate
from workloads import programs as P

HERE = os.path.dirname(os.path.abspath(__file__))


def run(prog, G, mode="auto", step=4):
    rt = Runtime(G, lookahead=mode, horizon_step=step)
    run_program(rt, prog)
    return rt


def bytes_match(rt, prog):
    res = simulate(rt)
    exp, mask = sequential(prog)
    return all((res[k][mask[k]] == exp[k][mask[k]]).all() for k in exp)


def ancestors(log):
    anc = []
    for rec in log:
        a = 0
        for d in rec["deps"]:
            a |= anc[d] | (1 << d)
        anc.append(a)
    return anc


# ------------------------------------------------------------ Fig. 4
def test_fig4_nbody_structure():
    gold = json.load(open(os.path.join(HERE, "golden", "fig4_nbody_g2.json")))
    N = 256
    prog = P.nbody(N, steps=2, host_init=True)
    rt = run(prog, gold["n_devices"])
    log = rt.log

    def frac(f):
        return [N * f[0][0] // f[0][1], N * f[1][0] // f[1][1]]

    allocs = [(r["buffer"], r["mem"], r["box"][0][0], r["box"][1][0]) for r in log if r["kind"] == "alloc"]
    exp = [(a["buffer"], a["mem"], *frac(a["box_frac"])) for a in gold["allocs"]]
    assert sorted(allocs) == sorted(exp)
    # first timestep (task 1): P and V made coherent from host memory M0
    t1 = [r for r in log if r["kind"] == "copy" and r["task"] == 1]
    assert len(t1) == 4 and all(r["src_mem"] == 0 for r in t1)
    # second timestep (task 3): exactly one pair of d2d copies
    t3 = [r for r in log if r["kind"] == "copy" and r["task"] == 3]
    got = sorted((r["buffer"], r["src_mem"], r["dst_mem"], r["region"][0][0][0], r["region"][0][1][0]) for r in t3)
    want = sorted((c["buffer"], c["src_mem"], c["dst_mem"], *frac(c["region_frac"])) for c in gold["second_timestep_d2d"])
    assert got == want
    # the two d2d copies are concurrent (no path between them)
    anc = ancestors(log)
    i, j = [r["iid"] for r in t3]
    assert not (anc[j] >> i) & 1 and not (anc[i] >> j) & 1
    # first horizon right after T4
    h = [r for r in log if r["kind"] == "horizon"]
    assert len(h) == 1 and h[0]["task"] == 5
    k4 = max(r["iid"] for r in log if r["kind"] == "kernel" and r["task"] == 4)
    assert (anc[h[0]["iid"]] >> k4) & 1
    assert bytes_match(rt, prog)
    check(log, rt.buf_meta, rt.tasks)


@pytest.mark.parametrize("G", [2, 3, 4, 8])
def test_nbody_allgather_copy_count(G):
    # every device needs every other device's chunk of P: G(G-1) d2d copies per step
    rt = run(P.nbody(64, steps=3, host_init=True), G)
    per_task = {}
    for r in rt.log:
        if r["kind"] == "copy" and r["src_mem"] >= 2 and r["dst_mem"] >= 2:
            per_task[r["task"]] = per_task.get(r["task"], 0) + 1
    assert sorted(per_task.values()) == [G * (G - 1)] * 2


# ------------------------------------------------------------ C1 table
def test_c1_counts_auto():
    rt = run(P.c1_chain(), 2, "auto")
    c = counts(rt.log)
    assert c == {"epoch": 3, "alloc": 4, "kernel": 8, "copy_d2d": 6, "horizon": 1, "copy_readback": 2, "free": 4}
    boxes = sorted((r["buffer"], r["mem"], r["box"][0][0], r["box"][1][0]) for r in rt.log if r["kind"] == "alloc")
    assert boxes == [(0, 2, 0, 2049), (0, 3, 2047, 4096), (1, 2, 0, 2049), (1, 3, 2047, 4096)]
    d2d = [(r["task"], r["buffer"], r["src_mem"], r["dst_mem"], r["region"]) for r in rt.log
           if r["kind"] == "copy" and r["reason"] == "coherence"]
    assert d2d[0] == (2, 0, 3, 2, [[[2048, 0, 0], [2049, 1, 1]]])
    assert d2d[1] == (2, 0, 2, 3, [[[2047, 0, 0], [2048, 1, 1]]])
    assert rt.flushes == 1            # only at the readback epoch


def test_c1_counts_none():
    rt = run(P.c1_chain(), 2, "none")
    c = counts(rt.log)
    assert c["alloc"] == 8 and c["copy_resize"] == 4 and c["free"] == 8
    assert c["copy_d2d"] == 6 and c["kernel"] == 8
    for r in rt.log:
        if r["kind"] == "copy" and r["reason"] == "resize":
            assert g.region_volume([((b[0][0], 0, 0), (b[1][0], 1, 1)) for b in r["region"]]) == 2048


def test_c1_required_edges():
    rt = run(P.c1_chain(), 2, "auto")
    log = rt.log
    anc = ancestors(log)
    k = {(r["task"], r["device"]): r["iid"] for r in log if r["kind"] == "kernel"}
    cp = [r for r in log if r["kind"] == "copy" and r["reason"] == "coherence"]
    # T3 kernel on D1 (writes A on M3) must follow the T2 halo copy reading A[2048] from M3
    c_t2_from_m3 = [r["iid"] for r in cp if r["task"] == 2 and r["src_mem"] == 3][0]
    assert (anc[k[(3, 1)]] >> c_t2_from_m3) & 1
    # T4 halo copy into M2's A[2048] must follow the T2 kernel on D0 that read that cell
    c_t4_to_m2 = [r["iid"] for r in cp if r["task"] == 4 and r["dst_mem"] == 2][0]
    assert (anc[c_t4_to_m2] >> k[(2, 0)]) & 1


# ------------------------------------------------------------ §4.3 lookahead
def test_listing5_resize_elision():
    prog = P.listing5(64)
    none = run(prog, 2, "none")
    auto = run(prog, 2, "auto")
    for m in (2, 3):
        na = [r for r in none.log if r["kind"] == "alloc" and r["mem"] == m and r["buffer"] == 0]
        nr = [r for r in none.log if r["kind"] == "copy" and r["reason"] == "resize" and r["dst_mem"] == m]
        assert len(na) >= 2 and len(nr) >= 1          # P:L562-563 "cause a resize allocation"
        aa = [r for r in auto.log if r["kind"] == "alloc" and r["mem"] == m and r["buffer"] == 0]
        assert len(aa) == 1
    assert counts(auto.log).get("copy_resize", 0) == 0
    assert bytes_match(none, prog) and bytes_match(auto, prog)


@pytest.mark.parametrize("G", [1, 2, 4])
def test_rsim_whole_program_queued(G):
    T, W = 24, 48
    prog = P.rsim(W, T)
    rt = Runtime(G, lookahead="auto")
    bids = [rt.buffer_create(b["dims"], b["extent"], b["elem_size"]) for b in prog["buffers"]]
    for op in prog["ops"]:
        if op[0] == "task":
            rt.task_submit(op[1])
    # "the entire command graph to be generated before the first instruction"
    assert len(rt.log) == 1
    rt.buffer_read(bids[0], P.full([T, W]))
    rt.shutdown()
    allocs = [(r["buffer"], r["mem"]) for r in rt.log if r["kind"] == "alloc"]
    assert sorted(allocs) == [(0, 2 + d) for d in range(G)]          # 1 per (buffer, memory)
    assert [r["box"] for r in rt.log if r["kind"] == "alloc"][0] == [[0, 0, 0], [T, W, 1]]
    assert rt.flushes == 1
    assert counts(rt.log).get("copy_resize", 0) == 0


def test_rsim_none_resizes_every_step():
    T, W = 16, 24
    rt = run(P.rsim(W, T), 2, "none")
    allocs = [r for r in rt.log if r["kind"] == "alloc" and r["mem"] == 2]
    assert len(allocs) == T
    assert bytes_match(rt, P.rsim(W, T))


def test_wavesim_flush_point():
    # R8: every step is non-allocating after step 2; the queue flushes on the 2nd
    # horizon after the last allocating command
    n = 32
    rt = Runtime(2, lookahead="auto")
    for b in P.wavesim(n, 0)["buffers"]:
        rt.buffer_create(b["dims"], b["extent"], b["elem_size"])
    for op in P.wavesim_init(n):
        rt.task_submit(op[1])
    k = 0
    while len(rt.log) == 1:
        rt.task_submit(P.wavesim_step(n, k)[1])
        k += 1
    assert k == 7                     # horizons after steps 3 and 7 (cp 4, 8)
    # steady state: no more queueing, no more allocs
    before = len([r for r in rt.log if r["kind"] == "alloc"])
    rt.task_submit(P.wavesim_step(n, k)[1])
    assert len([r for r in rt.log if r["kind"] == "alloc"]) == before
    assert rt.queue == []


def test_lookahead_transparency_and_monotone_benefit():
    for s in range(40):
        prog = P.random_program(1000 + s)
        for G in (1, 2, 3):
            res = {}
            for mode in ("none", "auto", "infinite"):
                rt = run(prog, G, mode)
                res[mode] = (simulate(rt), counts(rt.log).get("alloc", 0))
            exp, mask = sequential(prog)
            for mode in res:                       # S:L435 semantic transparency
                for k in exp:
                    assert (res[mode][0][k][mask[k]] == exp[k][mask[k]]).all()
            assert res["auto"][1] <= res["none"][1]


# ------------------------------------------------------------ horizons
def test_horizon_placement_linear_chain():
    n = 16
    rt = Runtime(1)
    rt.buffer_create(1, [n], 4)
    rt.task_submit({"dims": 1, "range": P.full([n]), "kernel": "probe", "params": {"salt": 0},
                    "accesses": [(0, "write", ("one_to_one",))]})
    for i in range(11):
        rt.task_submit({"dims": 1, "range": P.full([n]), "kernel": "probe", "params": {"salt": i},
                        "accesses": [(0, "read_write", ("one_to_one",))]})
    rt.wait()
    # tasks 1..12 form a chain; horizons after T4, T8, T12 get tids 5, 10, 15
    hs = [r["task"] for r in rt.log if r["kind"] == "horizon"]
    assert hs == [5, 10, 15]


def test_horizon_bounds_tracking():
    # AC5: 1000-iteration loop keeps tracker state bounded
    n = 32
    sizes = {}
    for step in (2, 4):
        rt = Runtime(2, horizon_step=step)
        for b in P.wavesim(n, 0)["buffers"]:
            rt.buffer_create(b["dims"], b["extent"], b["elem_size"])
        for op in P.wavesim_init(n):
            rt.task_submit(op[1])
        peak = 0
        for k in range(1000):
            rt.task_submit(P.wavesim_step(n, k)[1])
            vals = set()
            for buf in rt.bufs.values():
                vals |= set(buf.orig_writer.values())
                for lst in buf.live.values():
                    for a in lst:
                        vals |= set(a.last_writer.values())
                        for s in a.readers.values():
                            vals |= set(s)
            peak = max(peak, len(vals))
            if k == 100:
                early = peak
        assert peak == early           # no growth after the first 100 steps
        sizes[step] = peak
    assert sizes[4] >= sizes[2]


# ------------------------------------------------------------ §4.4 diagnostics
def test_overlapping_write_error():
    rt = Runtime(2)
    rt.buffer_create(1, [16], 4)
    log_len = len(rt.log)
    with pytest.raises(CelError) as e:       # P:L614 "a writing accessor with an all range mapper"
        rt.task_submit({"dims": 1, "range": P.full([16]), "kernel": "probe", "params": {"salt": 1},
                        "accesses": [(0, "write", ("all",))]})
    assert e.value.code == CelError.OVERLAPPING_WRITE
    assert len(rt.log) == log_len and rt.tdag.next_tid == 1       # state unchanged
    # neighborhood(1) writer split two ways overlaps on the boundary band
    with pytest.raises(CelError):
        rt.task_submit({"dims": 1, "range": P.full([16]), "kernel": "probe", "params": {"salt": 1},
                        "accesses": [(0, "write", ("neighborhood", (1,)))]})
    # one_to_one writer: fine
    assert rt.task_submit({"dims": 1, "range": P.full([16]), "kernel": "probe", "params": {"salt": 1},
                           "accesses": [(0, "write", ("one_to_one",))]})[1] == 0


def test_uninitialized_read_warning():
    rt = Runtime(2)
    rt.buffer_create(1, [16], 4)
    rt.buffer_create(1, [16], 4)
    rt.task_submit({"dims": 1, "range": ([0], [8]), "kernel": "probe", "params": {"salt": 1},
                    "accesses": [(0, "write", ("one_to_one",))]})
    tid, st = rt.task_submit({"dims": 1, "range": P.full([16]), "kernel": "probe", "params": {"salt": 2},
                              "accesses": [(0, "read", ("one_to_one",)), (1, "write", ("one_to_one",))]})
    assert st == 1                                                   # P:L607 warning
    assert rt.warnings[-1][2] == g.region(g.box([8], [16]))          # [n/2, n)
    rt.shutdown()
    check(rt.log, rt.buf_meta, rt.tasks)


# ------------------------------------------------------------ invariants
@pytest.mark.parametrize("G", [1, 2, 3, 4, 8])
def test_random_programs_semantics_and_invariants(G):
    for s in range(25):
        prog = P.random_program(100 * G + s)
        for mode in ("none", "auto"):
            rt = run(prog, G, mode, step=2 + s % 3)
            assert bytes_match(rt, prog)
            check(rt.log, rt.buf_meta, rt.tasks)


@pytest.mark.parametrize("prog,G", [(P.wavesim(24, 6), 4), (P.jacobi3d(10, 3), 8), (P.rsim(20, 10), 3),
                                    (P.nbody(40, 2), 4), (P.c1_chain(256), 2)])
def test_configs_small(prog, G):
    for mode in ("none", "auto"):
        rt = run(prog, G, mode)
        assert bytes_match(rt, prog)
        check(rt.log, rt.buf_meta, rt.tasks)


def test_checker_catches_mutations():
    """The checker itself must reject a log with a dropped copy or dependency."""
    prog = P.c1_chain(64)
    rt = run(prog, 2)
    base = rt.log
    check(base, rt.buf_meta, rt.tasks)
    # drop one coherence copy -> stale read
    i = [r["iid"] for r in base if r["kind"] == "copy" and r["reason"] == "coherence"][0]
    mutated = []
    for r in base:
        if r["iid"] == i:
            r = dict(r, kind="horizon")
        mutated.append(r)
    with pytest.raises(InvariantError):
        check(mutated, rt.buf_meta, rt.tasks)
    # drop a kernel's dataflow dependency on that copy -> RAW unordered
    for r in base:
        if r["kind"] == "kernel" and i in r["deps"]:
            mutated = [dict(x, deps=[d for d in x["deps"] if d != i]) if x["iid"] == r["iid"] else x for x in base]
            break
    with pytest.raises(InvariantError):
        check(mutated, rt.buf_meta, rt.tasks)


def test_allocation_checker_catches_mutations():
    """R9 pins: the checker itself must reject a log whose
    allocations overlap, shrink or leak."""
    from oracle.invariants import check_allocations
    prog = P.c1_chain(64)
    rt = run(prog, 2, "none")          # lookahead none: resize chains alloc -> copy -> free
    base = rt.log
    st = check_allocations(base)
    assert st["allocs"] == st["freed"] == 8
    chain = [r for r in base if r["kind"] == "copy" and r["reason"] == "resize"][0]
    new = next(r for r in base if r["kind"] == "alloc" and r["aid"] == chain["dst_aid"])
    old = next(r for r in base if r["kind"] == "alloc" and r["aid"] == chain["src_aid"])

    def mutate(fn):
        return [fn(dict(r)) for r in base]

    # shrunk: the replacing allocation no longer contains the one it replaces
    def shrink(r):
        if r["iid"] == new["iid"]:
            r["box"] = [list(old["box"][0]), [old["box"][1][0] - 1] + list(old["box"][1][1:])]
        return r
    with pytest.raises(InvariantError):
        check_allocations(mutate(shrink))
    # overlap: the old allocation is not freed at the end of its resize chain
    free_old = next(r for r in base if r["kind"] == "free" and r["aid"] == old["aid"])

    def keep_old(r):
        return dict(r, kind="horizon") if r["iid"] == free_old["iid"] else r
    with pytest.raises(InvariantError, match="overlap"):
        check_allocations(mutate(keep_old), closed=False)
    # overlap without containment: a fresh allocation straddling a live one
    extra = dict(new, aid=999, box=[[new["box"][1][0] - 1, 0, 0], [new["box"][1][0] + 1, 1, 1]])
    with pytest.raises(InvariantError, match="without containing"):
        check_allocations(base[:new["iid"] + 1] + [extra] + base[new["iid"] + 1:], closed=False)
    # leaked: a final free dropped
    last_free = [r for r in base if r["kind"] == "free"][-1]

    def leak(r):
        return dict(r, kind="horizon") if r["iid"] == last_free["iid"] else r
    with pytest.raises(InvariantError, match="never freed"):
        check_allocations(mutate(leak))
    # double free
    with pytest.raises(InvariantError):
        check_allocations(base + [dict(last_free, iid=len(base))])
