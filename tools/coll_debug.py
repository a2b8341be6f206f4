"""Two-process all-gather debug run: small N-body with the NCCL collective."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist
from paper_2503_10516_b200 import cel
from workloads import programs as P
import bench

rank, world, local = bench.env_rank()
dist.init_process_group("gloo")
torch.cuda.set_device(rank)
rt = bench.make_runtime(cel, world, rank, world, dist, 64 << 20)
print("rank", rank, "runtime up", flush=True)
prog = P.nbody(int(sys.argv[1]) if len(sys.argv) > 1 else 64, 1)
from workloads.driver import run_program
out = run_program(rt, prog)
print("rank", rank, "done", flush=True)
dist.barrier()
dist.destroy_process_group()
