"""The scheduler's steady-state compile memo (csrc/sched_memo.cpp) changes
nothing but host time: with it (default) and without it (CEL_SCHED_MEMO=0)
the C++ scheduler writes the same instruction log, record for record, and on
iterative programs that log is still the oracle's.  The memo must actually
replay (hits > 0) where the state is periodic (WaveSim, Jacobi, N-body), and
random programs whose task sequence repeats exercise hits from irregular
states (reads, waits and partial ranges in between)."""

import json
import os

import pytest

from oracle.invariants import check
from oracle.scheduler import Runtime as OracleRuntime
from workloads.driver import run_program
from workloads import programs as P


@pytest.fixture(scope="module")
def cel():
    import __graft_entry__
    __graft_entry__.build()
    from paper_2503_10516_b200 import cel as c
    return c


def cpp_log(cel, prog, G, mode, step, memo, monkeypatch, tmp):
    monkeypatch.setenv("CEL_SCHED_MEMO", "1" if memo else "0")
    r = cel.Runtime(G, execute=False, lookahead=mode, horizon_step=step, instr_log_path=tmp)
    st = {}

    def keep(rt=r, close=r.shutdown):
        if rt.h is not None:
            st.update(rt.stats())
        close()
    r.shutdown = keep
    run_program(r, prog)
    return [json.loads(line) for line in open(tmp)], st


def repeated(prog, times):
    """The program's task / read / wait sequence after its fills, `times` times."""
    ops = prog["ops"]
    k = 0
    while k < len(ops) and ops[k][0] == "task" and ops[k][1]["kernel"] in ("probe", "fill_hash") and \
            len(ops[k][1]["accesses"]) == 1 and ops[k][1]["accesses"][0][1] == "write":
        k += 1
    body = [op for op in ops[k:]]
    return dict(prog, ops=ops[:k] + body * times)


ITERATIVE = [
    ("wavesim", lambda: P.wavesim(48, 40)),
    ("wavesim2d", lambda: P.wavesim(40, 30, split="2d")),
    ("wavesim_axes", lambda: P.wavesim(40, 30, mapper="neighborhood_axes")),
    ("jacobi", lambda: P.jacobi3d(10, 16)),
    ("nbody", lambda: P.nbody(40, 12)),
    ("listing5", lambda: P.listing5(20)),
]


@pytest.mark.parametrize("name,make", ITERATIVE, ids=[n for n, _ in ITERATIVE])
@pytest.mark.parametrize("G", [1, 2, 3, 4, 8])
def test_memo_same_log_and_oracle(cel, monkeypatch, tmp_path, name, make, G):
    prog = make()
    for mode, step in (("auto", 4), ("none", 2), ("infinite", 3)):
        on, st_on = cpp_log(cel, prog, G, mode, step, True, monkeypatch, str(tmp_path / "on.jsonl"))
        off, st_off = cpp_log(cel, prog, G, mode, step, False, monkeypatch, str(tmp_path / "off.jsonl"))
        assert on == off
        assert st_off["memo_hits"] == 0
        for k in ("n_copy", "copies_coherence", "bytes_coherence", "bytes_d2d_peer", "gather_sets", "n_kernel"):
            assert st_on[k] == st_off[k], k
        if name != "listing5":
            assert st_on["memo_hits"] > 0, (name, G, mode)
    o = OracleRuntime(G, lookahead="auto", horizon_step=4)
    run_program(o, prog)
    on, _ = cpp_log(cel, prog, G, "auto", 4, True, monkeypatch, str(tmp_path / "on.jsonl"))
    assert o.log == on
    check(on, o.buf_meta, o.tasks)


@pytest.mark.parametrize("G", [1, 2, 4])
def test_memo_repeated_random_programs(cel, monkeypatch, tmp_path, G):
    hits = 0
    for s in range(24):
        prog = repeated(P.random_program(9100 + 13 * G + s, max_tasks=6), 5)
        for mode in ("auto", "none"):
            on, st = cpp_log(cel, prog, G, mode, 2 + s % 3, True, monkeypatch, str(tmp_path / "on.jsonl"))
            off, _ = cpp_log(cel, prog, G, mode, 2 + s % 3, False, monkeypatch, str(tmp_path / "off.jsonl"))
            assert on == off, (s, mode)
            hits += st["memo_hits"]
            if mode == "auto":
                o = OracleRuntime(G, lookahead="auto", horizon_step=2 + s % 3)
                run_program(o, prog)
                assert o.log == on
                check(on, o.buf_meta, o.tasks)
    assert hits > 0


def test_memo_full_size_wavesim_g8(cel, monkeypatch, tmp_path):
    """BASELINE size at G = 8: the memo serves every step after warm-up."""
    prog = P.wavesim(16384, 64)
    on, st = cpp_log(cel, prog, 8, "auto", 4, True, monkeypatch, str(tmp_path / "on.jsonl"))
    off, _ = cpp_log(cel, prog, 8, "auto", 4, False, monkeypatch, str(tmp_path / "off.jsonl"))
    assert on == off
    assert st["memo_hits"] >= 64 - 16
