"""GPU parity of virtual-node mode: N node schedulers and
executors in one process, exchanging data only through send / receive /
split receive / await receive instructions (M1 staging in pinned host memory,
pilots, receive arbitration by the Communicator).  Every readback must equal
the CPU oracle's byte simulation (oracle/cluster.py + simulate_cluster) bit for
bit, and every node's instruction log the oracle's."""

import json

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle.cluster import Cluster  # noqa: E402
from workloads.driver import run_program  # noqa: E402
from oracle.simulate import GARBAGE, simulate_cluster  # noqa: E402
from workloads import programs as P  # noqa: E402

LOG = "/tmp/cel_gpu_cluster.jsonl"


@pytest.fixture(scope="module")
def cel():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import __graft_entry__
    __graft_entry__.build()
    from paper_2503_10516_b200 import cel as c
    return c


def run_both(cel, prog, N, D, mode="auto", devices=None, step=4):
    devices = devices if devices is not None else [0] * (N * D)
    rt = cel.Runtime(D, cuda_devices=devices, lookahead=mode, horizon_step=step, arena_bytes=64 << 20,
                     instr_log_path=LOG, n_nodes=N)
    stats = {}
    close = rt.shutdown

    def keep():
        if rt.h is not None:
            stats.update(rt.stats())
        close()
    rt.shutdown = keep
    got = [r[1] for r in run_program(rt, prog) if r[0] == "read"]
    o = Cluster(N, D, lookahead=mode, horizon_step=step)
    run_program(o, prog)
    for k in range(N):
        assert [json.loads(line) for line in open("%s.%d" % (LOG, k))] == o.logs[k], "node %d log" % k
    exp = simulate_cluster(o)
    for k, arr in enumerate(got):
        defined = exp[k] != GARBAGE
        if not np.array_equal(arr[defined], exp[k][defined]):
            bad = np.argwhere((arr != exp[k]) & defined)
            raise AssertionError("readback %d: %d mismatches, first at %s" % (k, len(bad), bad[:3].tolist()))
    return stats


def test_fig4_nbody_two_nodes(cel):
    st = run_both(cel, P.nbody(256, 2, host_init=True), 2, 2)
    assert st["n_send"] > 0 and st["n_receive"] > 0 and st["pulls"] == st["n_send"]


@pytest.mark.parametrize("N,D", [(2, 1), (2, 2), (3, 1), (4, 1)])
def test_configs(cel, N, D):
    for prog in (P.c1_chain(256), P.wavesim(256, 7, rows=96), P.jacobi3d(20, 3), P.rsim(256, 12),
                 P.nbody(300, 2)):
        for mode in ("none", "auto"):
            run_both(cel, prog, N, D, mode)


def test_split_receive(cel):
    n = 4096
    prog = {"name": "split", "buffers": [{"dims": 1, "extent": [n], "elem_size": 4, "host_init": None},
                                         {"dims": 1, "extent": [n], "elem_size": 4, "host_init": None}],
            "ops": [P._task(1, P.full([n]), "fill_hash", [(0, "write", ("one_to_one",))], {"seed": 1}),
                    P._task(1, P.full([n]), "probe", [(0, "read", ("neighborhood", (1536,))),
                                                      (1, "write", ("one_to_one",))], {"salt": 3}),
                    ("read", 1, P.full([n]))]}
    st = run_both(cel, prog, 2, 2)
    assert st["n_split_receive"] > 0 and st["n_await_receive"] >= 2


@pytest.mark.parametrize("N,D", [(2, 1), (2, 2), (3, 2)])
def test_random_programs(cel, N, D):
    for s in range(10):
        prog = P.random_program(6100 + 11 * N + D + s)
        run_both(cel, prog, N, D, ["none", "auto", "infinite"][s % 3], step=2 + s % 3)


def test_nodes_on_distinct_gpus(cel):
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    for N, D in ((2, 1), (n, 1), (2, n // 2)):
        devs = list(range(N * D))
        for prog in (P.nbody(2048, 2), P.wavesim(1024, 5, rows=300), P.random_program(6200 + N)):
            run_both(cel, prog, N, D, devices=devs)


def test_degenerate_shapes(cel):
    """Nodes with empty command chunks, 1x1 grids, one-element buffers."""
    cases = [(P.wavesim(5, 3, rows=3), 4, 1), (P.wavesim(1, 3, rows=1), 2, 2), (P.nbody(1, 2), 2, 1),
             (P.nbody(3, 2), 2, 2), (P.jacobi3d(2, 2), 3, 1), (P.rsim(3, 4), 4, 1), (P.c1_chain(2), 3, 2)]
    for prog, N, D in cases:
        for mode in ("none", "auto"):
            run_both(cel, prog, N, D, mode)


@pytest.mark.parametrize("direct", [True, False])
def test_device_direct_sends(cel, direct, monkeypatch):
    """SURVEY NEXT-1 as written (the paper's RDMA future work; default
    in virtual-node mode, CEL_DIRECT_SENDS=0 turns it off): a push's staging
    copy into M1 is not executed; its
    sends publish the device allocation and the receiver pulls from it
    (NVLink between GPUs); a send spanning several devices' staged boxes, or
    any other use of the staged M1 bytes, executes the copies first.  Logs
    unchanged (the graph still has the staging copy), bytes bit-exact on the
    configs' stencil, N-body, RSim and 3-D programs (random programs: below)."""
    monkeypatch.setenv("CEL_DIRECT_SENDS", "1" if direct else "0")
    n = torch.cuda.device_count()
    devs2 = [0, 1 % n]
    for prog, N, D, devs in ((P.wavesim(1024, 7, rows=300), 2, 1, devs2), (P.nbody(2048, 2), 2, 1, devs2),
                             (P.nbody(512, 2, host_init=True), 2, 2, None), (P.wavesim(256, 7, rows=96), 2, 2, None),
                             (P.jacobi3d(20, 3), 2, 2, None), (P.rsim(256, 12), 2, 1, None)):
        st = run_both(cel, prog, N, D, devices=devs)
        if direct:
            assert st["staging_elided"] > st["staging_materialized"], (prog["name"], st["staging_elided"])
        else:
            assert st["staging_elided"] == 0


def test_device_direct_sends_random(cel, monkeypatch):
    """Device-direct sends on random programs (fixed / all / neighbourhood
    mappers, waits, readbacks, destroys, host data), where horizons subsume
    the staging copies' dependencies: bytes bit-exact."""
    monkeypatch.setenv("CEL_DIRECT_SENDS", "1")
    for s in range(10):
        run_both(cel, P.random_program(6400 + s), 2 + s % 2, 1 + s % 2, ["none", "auto", "infinite"][s % 3],
                 step=2 + s % 3)
