"""Pins for oracle/cluster.py (virtual-node mode): Fig. 4's
send / receive structure (tests/golden/fig4_nbody_2x2.json), the consumer
split of §3.4, SPMD consistency of pushes and pilots, the degenerate single
node, and semantic transparency against the plain sequential definition on
random programs over several topologies."""

import json
import os

import numpy as np
import pytest

from oracle import geometry as g
from oracle.cluster import Cluster
from oracle.invariants import check_allocations
from oracle.scheduler import Runtime
from workloads.driver import run_program
from oracle.simulate import sequential, simulate_cluster
from workloads import programs as P

HERE = os.path.dirname(os.path.abspath(__file__))


def run(prog, N, D, mode="auto", step=4):
    cl = Cluster(N, D, lookahead=mode, horizon_step=step)
    run_program(cl, prog)
    return cl


def bytes_match(cl, prog):
    res = simulate_cluster(cl)
    exp, mask = sequential(prog)
    return all(np.array_equal(res[k][mask[k]], exp[k][mask[k]]) for k in exp)


def ancestors(log):
    anc = []
    for rec in log:
        a = 0
        for d in rec["deps"]:
            a |= anc[d] | (1 << d)
        anc.append(a)
    return anc


def test_fig4_send_receive_structure():
    gold = json.load(open(os.path.join(HERE, "golden", "fig4_nbody_2x2.json")))
    N = 256
    prog = P.nbody(N, steps=2, host_init=True)
    cl = run(prog, gold["n_nodes"], gold["devices_per_node"])
    log = cl.logs[gold["node"]]
    t = [r for r in log if r["task"] == gold["task"]]

    def frac(f):
        return [N * f[0][0] // f[0][1], N * f[1][0] // f[1][1]]

    sends = [r for r in t if r["kind"] == "send"]
    assert len(sends) == gold["sends"]
    assert sorted([r["box"][0][0], r["box"][1][0]] for r in sends) == [frac(f) for f in gold["send_boxes_frac"]]
    assert all(r["target"] == gold["send_target"] and r["src_mem"] == 1 for r in sends)
    # each send depends only on its own device-to-host staging copy (and the M1 allocation)
    by_iid = {r["iid"]: r for r in log}
    for s in sends:
        stag = [by_iid[d] for d in s["deps"] if by_iid[d]["kind"] == "copy"]
        assert len(stag) == 1 and stag[0]["src_mem"] >= 2 and stag[0]["dst_mem"] == 1
        assert stag[0]["region"] == [s["box"]]
        assert all(by_iid[d]["kind"] in ("copy", "alloc") for d in s["deps"])
    assert len({d for s in sends for d in s["deps"] if by_iid[d]["kind"] == "copy"}) == gold["d2h_staging_copies"]
    # one pilot per send, addressed to the peer, with the send's box
    pil = [p for p in cl.nodes[0].pilots if p["transfer"][0] == gold["task"]]
    assert sorted(p["msg"] for p in pil) == sorted(s["msg"] for s in sends)
    assert all(p["receiver"] == gold["send_target"] for p in pil)
    recv = [r for r in t if r["kind"] in ("receive", "split_receive", "await_receive")]
    assert len(recv) == gold["receives"] and recv[0]["kind"] == "receive"
    assert recv[0]["region"] == [[[frac(gold["receive_region_frac"])[0], 0, 0], [frac(gold["receive_region_frac"])[1], 1, 1]]]
    copies = [r for r in t if r["kind"] == "copy"]
    d2d = [r for r in copies if r["src_mem"] >= 2 and r["dst_mem"] >= 2]
    from_m1 = [r for r in copies if r["src_mem"] == 1 and r["dst_mem"] >= 2]
    assert len(d2d) == gold["d2d_copies"] and len(from_m1) == gold["h2d_from_receive"]
    assert all(recv[0]["iid"] in r["deps"] for r in from_m1)
    # Fig. 4 caption: every send and receive is concurrent with the others
    anc = ancestors(log)
    xs = [r["iid"] for r in sends + recv]
    for i in xs:
        for j in xs:
            assert i == j or not (anc[j] >> i) & 1
    assert [r["task"] for r in log if r["kind"] == "horizon"] == [gold["horizon_task"]]
    assert bytes_match(cl, prog)


def test_consumer_split_await_receives():
    """§3.4: consumers reading different parts of the awaited
    region -> split receive + one await receive per consumer-split fragment;
    each consumer depends on the await receives covering its input."""
    n = 16
    prog = {"name": "split", "buffers": [{"dims": 1, "extent": [n], "elem_size": 4, "host_init": None},
                                         {"dims": 1, "extent": [n], "elem_size": 4, "host_init": None}],
            "ops": [P._task(1, P.full([n]), "fill_hash", [(0, "write", ("one_to_one",))], {"seed": 1}),
                    P._task(1, P.full([n]), "probe", [(0, "read", ("neighborhood", (6,))),
                                                      (1, "write", ("one_to_one",))], {"salt": 3}),
                    ("read", 1, P.full([n]))]}
    cl = run(prog, 2, 2)
    log = cl.logs[0]
    sr = [r for r in log if r["kind"] == "split_receive"]
    aw = [r for r in log if r["kind"] == "await_receive"]
    assert len(sr) == 1 and sr[0]["region"] == [[[8, 0, 0], [14, 1, 1]]]
    # device 0 ([0,4)) reads [0,10), device 1 ([4,8)) reads [0,14): atoms [8,10) and [10,14)
    assert [r["region"] for r in aw] == [[[[8, 0, 0], [10, 1, 1]]], [[[10, 0, 0], [14, 1, 1]]]]
    assert all(r["deps"] == [sr[0]["iid"]] for r in aw)
    assert bytes_match(cl, prog)


def test_pushes_match_awaits_and_pilots():
    """SPMD consistency: per (receiver, transfer) the senders' pilot
    boxes are disjoint and tile the receiver's receive region exactly."""
    for seed in range(20):
        prog = P.random_program(4100 + seed)
        cl = run(prog, 3, 2, ["none", "auto"][seed % 2])
        pil = cl.pilots()
        for n, log in enumerate(cl.logs):
            for r in log:
                if r["kind"] not in ("receive", "split_receive"):
                    continue
                tr = tuple(r["transfer"])
                boxes = [p["box"] for p in pil if p["receiver"] == n and tuple(p["transfer"]) == tr]
                reg = tuple((tuple(b[0]), tuple(b[1])) for b in r["region"])
                assert g.region_volume(g.region_union(*[(b,) for b in boxes])) == sum(g.volume(b) for b in boxes)
                assert g.region_union(*[(b,) for b in boxes]) == g.canon(list(reg))
        assert bytes_match(cl, prog)


def test_single_node_is_the_single_node_runtime():
    for seed in range(10):
        prog = P.random_program(4200 + seed)
        cl = run(prog, 1, 3)
        rt = Runtime(3)
        run_program(rt, prog)
        assert cl.logs[0] == rt.log


@pytest.mark.parametrize("N,D", [(2, 1), (2, 2), (3, 1), (3, 2), (4, 1)])
def test_random_programs_match_sequential(N, D):
    for s in range(25):
        prog = P.random_program(4300 + 31 * N + 7 * D + s)
        cl = run(prog, N, D, ["none", "auto", "infinite"][s % 3], step=2 + s % 3)
        assert bytes_match(cl, prog), s
        for log in cl.logs:                 # R9 per node, M1 staging allocations included
            check_allocations(log)


@pytest.mark.parametrize("N,D", [(2, 2), (4, 1)])
def test_configs_match_sequential(N, D):
    for prog in (P.c1_chain(64), P.wavesim(64, 5, rows=40), P.jacobi3d(12, 3), P.rsim(64, 10),
                 P.nbody(100, 2), P.nbody(64, 2, host_init=True)):
        for mode in ("none", "auto"):
            cl = run(prog, N, D, mode)
            assert bytes_match(cl, prog), (prog["name"], mode)
            for log in cl.logs:
                check_allocations(log)


def pushed_elements(cl):
    return sum(g.volume(p["box"]) for p in cl.pilots())


@pytest.mark.parametrize("N,D", [(2, 1), (3, 2), (4, 1), (4, 2)])
@pytest.mark.parametrize("mapper", ["neighborhood", "neighborhood_axes"])
def test_wavesim_halo_volume_closed_form(N, D, mapper):
    """Closed form of the inter-node traffic of a radius-1 stencil under the
    1-D node split (§3.4 push / await-push; R17): every step each
    of the N-1 interior boundaries exchanges one full row each way
    (2(N-1) rows of n cells; the buffer read was rewritten by its owners in the
    previous step, so no halo is still valid), the devices inside a node
    add nothing, and the final readback of both buffers makes node 0 pull the
    R - R/N rows it does not own, twice, less the one halo row of the buffer
    the last step read, which node 0 received then and still holds (R17
    holders: not rewritten since)."""
    R, n, steps = 6 * N, 10, 3
    cl = run(P.wavesim(n, steps, rows=R, mapper=mapper), N, D)
    assert pushed_elements(cl) == steps * 2 * (N - 1) * n + (2 * (R - R // N) - 1) * n
    # every step push is one row, from an adjacent node
    for p in cl.pilots():
        (lo, hi) = p["box"]
        if hi[0] - lo[0] == 1:
            assert abs(p["sender"] - p["receiver"]) == 1


@pytest.mark.parametrize("N", [2, 3, 4])
@pytest.mark.parametrize("host_init", [False, True])
def test_nbody_allgather_volume_closed_form(N, host_init):
    """Closed form for the all-gather of Listing 1 ("all" mapper):
    a timestep makes every node receive the n - n/N bodies it does not own,
    (N-1) n in total, except the first one when the positions are host data
    present on every node (R17 ALL); the readback of P and V pulls n - n/N
    bodies of each to node 0."""
    n, steps = 12 * N, 3
    cl = run(P.nbody(n, steps, host_init=host_init), N, 1)
    gathers = steps - (1 if host_init else 0)
    assert pushed_elements(cl) == gathers * (N - 1) * n + 2 * (n - n // N)
