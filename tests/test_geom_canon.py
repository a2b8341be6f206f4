"""Region canonical form (R2): the scheduler's stack-only path for
boxes that share one dim-2 range (csrc/geom.hpp detail::canon_2d) produces
exactly the general maximal-slab dissection (detail::canon_dim) -- random
regions, compiled with the host compiler (no GPU)."""

import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_canon_2d_equals_general_dissection(tmp_path):
    gxx = shutil.which("g++")
    if not gxx:
        pytest.skip("no g++")
    exe = str(tmp_path / "canon_2d_test")
    subprocess.run([gxx, "-O2", "-std=c++17", "-I", os.path.join(ROOT, "paper_2503_10516_b200", "csrc"),
                    os.path.join(ROOT, "tests", "cpp", "canon_2d_test.cpp"), "-o", exe], check=True)
    r = subprocess.run([exe], stdout=subprocess.PIPE, timeout=300)
    assert r.returncode == 0, r.stdout.decode()
    assert r.stdout.decode().startswith("0 / ")
