"""N>1 path: one process per device (torchrun).  CPU: world-size-2 gloo run of
the replicated scheduler (execute=0) — every rank's instruction log equals the
oracle's.  GPU: the same programs executed with peer pushes over NVLink and
cross-process flag waits, readbacks merged and compared bit-exactly."""

import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def torchrun(n, *args, port=29533, timeout=600, extra_env=None):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(n),
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "tests", "mp_check.py")]
    cmd += list(args)
    env = dict(os.environ, OMP_NUM_THREADS="1", CEL_COLL_MIN_BYTES="0")   # exercise the NCCL gathers
    env.update(extra_env or {})
    return subprocess.run(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, timeout=timeout, env=env, cwd=ROOT)


@pytest.mark.parametrize("world", [2, 4])
def test_replicated_scheduler_gloo(world):
    import __graft_entry__
    __graft_entry__.build()
    r = torchrun(world, "--execute", "0", "--quick", port=29533 + world)
    out = r.stdout.decode()
    assert r.returncode == 0 and "MP_CHECK PASS" in out, out[-3000:]


@pytest.mark.gpu
def test_multiprocess_gpu():
    """One process per GPU; on a one-GPU box two ranks share it (--fold 1):
    the IPC-mapped arenas, cross-process flag waits and the rank filter run
    the same way, only the pushes stay inside one HBM (no NCCL: it needs
    distinct GPUs)."""
    torch = pytest.importorskip("torch")
    n = torch.cuda.device_count()
    if n < 1:
        pytest.skip("needs a GPU")
    if n >= 2:
        r = torchrun(min(n, 4), "--execute", "1", port=29534)
    else:
        r = torchrun(2, "--execute", "1", "--fold", "1", port=29536, timeout=900)
    out = r.stdout.decode()
    assert r.returncode == 0 and "MP_CHECK PASS" in out, out[-3000:]


@pytest.mark.gpu
@pytest.mark.parametrize("fuse", ["1", "0"])
def test_multiprocess_halo_fused(fuse):
    """WaveSim's halo exchange fused into the stencil launches (exec_halo.cu,
    CEL_FUSE_HALO, on by default): ranks on distinct GPUs push boundary rows from the
    computing CTAs into the neighbours' memory and await incoming rows in the
    reading CTAs; the readbacks equal the oracle's bytes and the instruction
    logs its log, with the fused path taken (or, fuse=0, not)."""
    torch = pytest.importorskip("torch")
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs two GPUs (in-kernel flag waits across processes sharing a GPU are unsafe)")
    r = torchrun(min(n, 4), "--execute", "1", "--quick", "--only", "wavesim", port=29540 + int(fuse),
                 extra_env={"CEL_FUSE_HALO": fuse})
    out = r.stdout.decode()
    assert r.returncode == 0 and "MP_CHECK PASS" in out, out[-3000:]
    assert ("halo copies fused" in out) == (fuse == "1"), out[-3000:]
