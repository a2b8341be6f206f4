"""One resize copy through the C-ABI (for ncu captures of the copy kernels):
  python tools/copy_case.py 2d|3d|1g     (CEL_COPY=tma selects the TMA tensor-map kernel)
2d: 8192 x 16 KiB rows at a 16 KiB pitch into a 16400 B pitch; 3d: 256 x 64 x
4 KiB; 1g: 1 GiB contiguous.  Runs the case twice (the second is the one to
profile: launch-skip the first)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["CEL_NO_GROW"] = "1"
from paper_2503_10516_b200 import cel  # noqa: E402

case = sys.argv[1] if len(sys.argv) > 1 else "2d"
shapes = {"2d": ([8192, 16384], [8192, 4096], ([0, 4095], [8192, 4097])),
          "3d": ([256, 80, 1024], [256, 64, 1024], ([0, 63, 0], [256, 65, 1024])),
          "1g": ([(1 << 28) + 1], [1 << 28], ([(1 << 28) - 1], [(1 << 28) + 1]))}
ext, written, fixed = shapes[case]
for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 2):
    rt = cel.Runtime(1, lookahead="none", arena_bytes=3 << 30)
    d = len(ext)
    rt.buffer_create(d, ext, 4)
    rt.task_submit({"dims": d, "range": ([0] * d, written), "kernel": "fill_hash", "params": {"seed": 11},
                    "accesses": [(0, "write", ("one_to_one",))]})
    rt.wait()
    rt.profile_enable(True)
    rt.task_submit({"dims": 1, "range": ([0], [1]), "kernel": "fill_const", "params": {"value": 2.0},
                    "accesses": [(0, "write", ("fixed", fixed))]})
    rt.wait()
    ms, cnt = rt.profile_read().get("copy", (0.0, 0))
    st = rt.stats()
    print(case, st["copies_resize"], "resize copies,", st["tma_copy_launches"], "TMA launches, %.1f us, %.3f TB/s rw"
          % (ms * 1e3, 2 * st["bytes_resize"] / (ms / 1e3) / 1e12 if ms else 0))
    rt.shutdown()
