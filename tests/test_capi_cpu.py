"""CPU tests of the C-ABI library (no GPU): it loads, exports every symbol
include/cel.h declares, and its scheduler (execute=0: instruction graph only,
no CUDA call) produces exactly the oracle's instruction log — record for
record, dependencies included — on every config and on random programs."""

import json
import os
import re

import pytest

from oracle.invariants import check
from oracle.scheduler import Runtime as OracleRuntime
from workloads.driver import run_program
from workloads import programs as P

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def cel():
    import __graft_entry__
    __graft_entry__.build()
    from paper_2503_10516_b200 import cel as c
    return c


def header_functions():
    src = open(os.path.join(ROOT, "include", "cel.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:int|size_t|const char\*)\s+(cel_\w+)\s*\(", src, flags=re.M)))


def test_library_exports_every_declared_symbol(cel):
    names = header_functions()
    assert len(names) >= 14
    for n in names:
        assert hasattr(cel.lib, n), n
    assert sorted(cel.SYMBOLS) == names


def test_no_gpu_means_loud_failure(cel):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(cel.CelError) as e:
        cel.Runtime(1, execute=True)
    assert e.value.code == cel.E_CUDA


def both_logs(cel, prog, G, mode, step=4, tmp="/tmp/cel_cpu_log.jsonl"):
    o = OracleRuntime(G, lookahead=mode, horizon_step=step)
    run_program(o, prog)
    r = cel.Runtime(G, execute=False, lookahead=mode, horizon_step=step, instr_log_path=tmp)
    run_program(r, prog)
    c = [json.loads(line) for line in open(tmp)]
    return o, c


def assert_same(o, c):
    assert len(o.log) == len(c)
    for a, b in zip(o.log, c):
        assert a == b


@pytest.mark.parametrize("G", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("mode", ["none", "auto", "infinite"])
def test_config_logs_match_oracle(cel, G, mode):
    for prog in (P.c1_chain(), P.wavesim(48, 9), P.nbody(40, 3, host_init=True), P.nbody(40, 2),
                 P.rsim(30, 12), P.jacobi3d(10, 3), P.listing5(20)):
        o, c = both_logs(cel, prog, G, mode)
        assert_same(o, c)
        check(c, o.buf_meta, o.tasks)          # the C++ graph passes the brute-force checker


@pytest.mark.parametrize("G", [1, 2, 3, 4, 8])
def test_random_logs_match_oracle(cel, G):
    for s in range(30):
        prog = P.random_program(7000 + 31 * G + s)
        for mode in ("none", "auto"):
            o, c = both_logs(cel, prog, G, mode, step=2 + s % 3)
            assert_same(o, c)


def test_full_size_instruction_counts(cel):
    """Instruction parity at BASELINE sizes (execute=0 is cheap: regions only)."""
    for prog, G in ((P.wavesim(16384, 12), 8), (P.jacobi3d(1024, 4), 8), (P.nbody(1 << 20, 3), 8),
                    (P.c1_chain(), 2)):
        o, c = both_logs(cel, prog, G, "auto")
        assert_same(o, c)


def test_rsim_full_size_lookahead(cel):
    """Config 4 at W=84,000, T=256: auto allocates once per memory, none resizes every step."""
    prog = P.rsim(84000, 256)
    o, c = both_logs(cel, prog, 4, "auto")
    assert_same(o, c)
    assert sum(1 for r in c if r["kind"] == "alloc") == 4
    o, c = both_logs(cel, prog, 4, "none")
    assert_same(o, c)
    assert sum(1 for r in c if r["kind"] == "alloc") == 4 * 256


def _gather_sets(cel, prog, G):
    rt = cel.Runtime(G, execute=False)
    st = {}

    def keep(rt=rt, close=rt.shutdown):
        if rt.h is not None:
            st.update(rt.stats())
        close()
    rt.shutdown = keep
    run_program(rt, prog)
    return st["gather_sets"], st["copies_coherence"]


def test_all_gather_detection(cel, monkeypatch):
    """§8 a7: coherence copy sets of a buffer read through `all` / `fixed`
    mappers, where every device receives each other device's one contiguous
    chunk, are flagged as all-gathers; neighbourhood halos never are."""
    monkeypatch.setenv("CEL_COLL_MIN_BYTES", "0")
    for G in (2, 3, 4):
        assert _gather_sets(cel, P.nbody(1000, 2), G) == (2, 2 * G * (G - 1))
        assert _gather_sets(cel, P.rsim(1000, 8), G) == (7, 7 * G * (G - 1))
        assert _gather_sets(cel, P.wavesim(256, 4, rows=64), G)[0] == 0
        assert _gather_sets(cel, P.jacobi3d(16, 2), G)[0] == 0
        assert _gather_sets(cel, P.c1_chain(64), G)[0] == 0
    assert _gather_sets(cel, P.nbody(1000, 2), 1) == (0, 0)
    # a 2-D buffer gathered in multi-row boxes is not flagged: the executor pads
    # allocation rows to 16 bytes, so such boxes need not be one byte run
    n = 64
    prog = {"name": "all2d", "buffers": [{"dims": 2, "extent": [n, n], "elem_size": 4, "host_init": None},
                                         {"dims": 2, "extent": [n, n], "elem_size": 4, "host_init": None}],
            "ops": [P._task(2, P.full([n, n]), "fill_hash", [(0, "write", ("one_to_one",))], {"seed": 1}),
                    P._task(2, P.full([n, n]), "probe", [(0, "read", ("all",)), (1, "write", ("one_to_one",))],
                            {"salt": 2})]}
    for G in (2, 4):
        assert _gather_sets(cel, prog, G)[0] == 0
    # the default threshold (1 MiB per source) keeps small gathers on peer pushes
    monkeypatch.delenv("CEL_COLL_MIN_BYTES")
    assert _gather_sets(cel, P.nbody(1000, 2), 4)[0] == 0
    assert _gather_sets(cel, P.rsim(84000, 8), 4)[0] == 0
    assert _gather_sets(cel, P.nbody(1 << 20, 2), 4)[0] == 2


def test_errors_and_warnings(cel):
    r = cel.Runtime(2, execute=False)
    a = r.buffer_create(1, [16], 4)
    b = r.buffer_create(1, [16], 4)
    full = ([0], [16])
    with pytest.raises(cel.CelError) as e:       # writing accessor with an all mapper
        r.task_submit({"dims": 1, "range": full, "kernel": "probe", "params": {"salt": 1},
                       "accesses": [(a, "write", ("all",))]})
    assert e.value.code == cel.E_OVERLAPPING_WRITE
    with pytest.raises(cel.CelError) as e:
        r.task_submit({"dims": 1, "range": ([0], [20]), "kernel": "probe", "params": {"salt": 1},
                       "accesses": [(a, "write", ("one_to_one",))]})
    assert e.value.code == cel.E_OUT_OF_BOUNDS
    with pytest.raises(cel.CelError) as e:
        r.task_submit({"dims": 1, "range": full, "kernel": "probe", "params": {"salt": 1},
                       "accesses": [(a, "read", ("fixed", ([0], [40])))]})
    assert e.value.code == cel.E_OUT_OF_BOUNDS
    with pytest.raises(cel.CelError) as e:
        r.task_submit({"dims": 1, "range": full, "kernel": "probe", "params": {"salt": 1},
                       "accesses": [(99, "write", ("one_to_one",))]})
    assert e.value.code == cel.E_INVALID
    # rejected tasks left no trace: the first accepted task is tid 1
    tid, st = r.task_submit({"dims": 1, "range": ([0], [8]), "kernel": "probe", "params": {"salt": 1},
                             "accesses": [(a, "write", ("one_to_one",))]})
    assert (tid, st) == (1, 0)
    tid, st = r.task_submit({"dims": 1, "range": full, "kernel": "probe", "params": {"salt": 2},
                             "accesses": [(a, "read", ("one_to_one",)), (b, "write", ("one_to_one",))]})
    assert st == cel.W_UNINIT_READ
    r.buffer_destroy(a)
    with pytest.raises(cel.CelError):
        r.task_submit({"dims": 1, "range": full, "kernel": "probe", "params": {"salt": 3},
                       "accesses": [(a, "write", ("one_to_one",))]})
    r.shutdown()


# ------------------------------------------------------------ virtual-node mode
def cluster_logs(cel, prog, N, D, mode, step=4, tmp="/tmp/cel_cpu_cluster.jsonl"):
    from oracle.cluster import Cluster
    o = Cluster(N, D, lookahead=mode, horizon_step=step)
    run_program(o, prog)
    r = cel.Runtime(D, execute=False, lookahead=mode, horizon_step=step, instr_log_path=tmp, n_nodes=N)
    run_program(r, prog)
    return o, [[json.loads(line) for line in open("%s.%d" % (tmp, k))] for k in range(N)]


@pytest.mark.parametrize("N,D", [(2, 1), (2, 2), (3, 2), (4, 1)])
def test_cluster_config_logs_match_oracle(cel, N, D):
    for prog in (P.c1_chain(64), P.wavesim(64, 5, rows=40), P.jacobi3d(12, 3), P.rsim(64, 10), P.nbody(100, 2),
                 P.nbody(256, 2, host_init=True)):
        for mode in ("none", "auto"):
            o, c = cluster_logs(cel, prog, N, D, mode)
            for k in range(N):
                assert c[k] == o.logs[k], (prog["name"], mode, k)


@pytest.mark.parametrize("N,D", [(2, 1), (2, 2), (3, 1), (3, 2)])
def test_cluster_random_logs_match_oracle(cel, N, D):
    for s in range(20):
        prog = P.random_program(5100 + 13 * N + D + s)
        mode = ["none", "auto", "infinite"][s % 3]
        o, c = cluster_logs(cel, prog, N, D, mode, step=2 + s % 3)
        for k in range(N):
            assert c[k] == o.logs[k], (s, k)


def test_cluster_full_size_counts(cel):
    """N-body 2^20 on 2 nodes x 4 devices and WaveSim 16384^2 on 4 nodes x 2:
    instruction logs equal at BASELINE sizes (execute=0)."""
    for prog, N, D in ((P.nbody(1 << 20, 2), 2, 4), (P.wavesim(16384, 6), 4, 2)):
        o, c = cluster_logs(cel, prog, N, D, "auto")
        for k in range(N):
            assert c[k] == o.logs[k]
        assert sum(1 for r in c[0] if r["kind"] == "send") > 0


def test_axis_neighborhood_and_2d_wavesim_logs(cel):
    """WaveSim with the axis-only neighbourhood and the 2-D split:
    C++ logs equal the oracle's, and no corner element is ever copied."""
    for G in (2, 4, 6, 8):
        for split in ("1d", "2d"):
            prog = P.wavesim(96, 5, rows=72, split=split, mapper="neighborhood_axes")
            for mode in ("none", "auto"):
                o, c = both_logs(cel, prog, G, mode)
                assert_same(o, c)
                check(c, o.buf_meta, o.tasks)
    # 2-D split, 4 devices: the box neighbourhood also moves the 4 corner elements per step
    box = both_logs(cel, P.wavesim(96, 4, rows=72, split="2d"), 4, "auto")[1]
    axes = both_logs(cel, P.wavesim(96, 4, rows=72, split="2d", mapper="neighborhood_axes"), 4, "auto")[1]
    ncopy = lambda log: sum(1 for r in log if r["kind"] == "copy" and r["reason"] == "coherence")  # noqa: E731
    assert ncopy(box) - ncopy(axes) == 4 * 4


def degenerate_cases():
    """Fewer rows / bodies / cells than devices (empty chunks, R4), 1x1 grids,
    one-element buffers, 2-D split on a 2x4 grid."""
    return [(P.wavesim(5, 3, rows=3), 4), (P.wavesim(1, 3, rows=1), 2), (P.nbody(1, 2), 2), (P.nbody(3, 2), 4),
            (P.jacobi3d(2, 2), 3), (P.rsim(3, 4), 4), (P.c1_chain(2), 4),
            (P.wavesim(4, 2, rows=2, split="2d", mapper="neighborhood_axes"), 4)]


@pytest.mark.parametrize("mode", ["none", "auto"])
def test_degenerate_shapes_logs_match_oracle(cel, mode):
    for prog, G in degenerate_cases():
        o, c = both_logs(cel, prog, G, mode)
        assert_same(o, c)
        check(c, o.buf_meta, o.tasks)          # and the brute-force checker


def test_cluster_degenerate_shapes(cel):
    """More nodes than rows / bodies (nodes with empty command chunks, R17
    1-D node split), 1x1 grids and one-element buffers: every node's C++ log
    equals the oracle's and the oracle's bytes equal the sequential definition."""
    import numpy as np
    from oracle.simulate import sequential, simulate_cluster
    cases = [(P.wavesim(5, 3, rows=3), 4, 1), (P.wavesim(1, 3, rows=1), 2, 2), (P.nbody(1, 2), 2, 1),
             (P.nbody(3, 2), 2, 2), (P.jacobi3d(2, 2), 3, 1), (P.rsim(3, 4), 4, 1), (P.c1_chain(2), 3, 2)]
    for prog, N, D in cases:
        for mode in ("none", "auto"):
            o, c = cluster_logs(cel, prog, N, D, mode)
            assert c == o.logs
            res = simulate_cluster(o)
            exp, mask = sequential(prog)
            assert all(np.array_equal(res[k][mask[k]], exp[k][mask[k]]) for k in exp)
