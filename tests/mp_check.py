"""Multi-process parity (one process per GPU, torchrun): every rank runs the
replicated scheduler, executes the instructions of its own device, pushes
coherence copies into peer GPUs' memory over NVLink and orders cross-process
dependencies with stream memory-op flags.  Readbacks from all ranks are
merged and compared bit-exactly with the CPU oracle; the instruction log of
every rank must equal the oracle's.

  torchrun --nproc-per-node N --master-addr 127.0.0.1 tests/mp_check.py [--execute 0]
"""

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch.distributed as dist  # noqa: E402

from oracle.scheduler import Runtime as OracleRuntime  # noqa: E402
from workloads.driver import run_program  # noqa: E402
from oracle.simulate import GARBAGE, simulate  # noqa: E402
from workloads import programs as P  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--execute", type=int, default=1)
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--only", default=None)
    ap.add_argument("--modes", default="auto,none")
    ap.add_argument("--fold", type=int, default=0,
                    help="k > 0: ranks share k GPUs (rank r on GPU r %% k): CUDA IPC and flags within one GPU")
    args = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dist.init_process_group("gloo")
    from paper_2503_10516_b200 import cel
    progs = [P.c1_chain(4096), P.wavesim(1024, 9, rows=700), P.nbody(3000, 2), P.nbody(500, 2, host_init=True),
             P.rsim(3000, 20), P.jacobi3d(40, 3)]
    w2 = P.wavesim(512, 7, rows=300, split="2d", mapper="neighborhood_axes")
    w2["name"] = "wavesim2d"
    progs.append(w2)
    modes = args.modes.split(",")
    if args.only:
        progs = [p for p in progs if p["name"] == args.only]
    if not args.quick:
        progs += [P.random_program(300 + s) for s in range(12)]
    nfail = 0
    for pi, prog in enumerate(progs):
        for mode in modes:
            log = "/tmp/mp_log_%d.jsonl" % rank
            if args.execute:
                import torch
                gpus = [r % args.fold if args.fold else r for r in range(world)]
                torch.cuda.set_device(gpus[rank])
                rt = cel.Runtime(world, cuda_devices=gpus, rank=rank, world=world,
                                 arena_bytes=256 << 20, lookahead=mode, instr_log_path=log)
                blobs = [None] * world
                dist.all_gather_object(blobs, rt.ipc_export())
                for r, b in enumerate(blobs):
                    if r != rank:
                        rt.ipc_import(r, b)
                dist.barrier()
                # readbacks land only where this rank's device holds the data: start from garbage
                orig = rt.buffer_read

                def read_garbage(bid, box, out=None, orig=orig):
                    dims, ext, es = rt.meta[bid]
                    mn = list(box[0]) + [0] * (3 - len(box[0]))
                    mx = list(box[1]) + [1] * (3 - len(box[1]))
                    shape = tuple(mx[d] - mn[d] for d in range(3)) + (es // 4,)
                    return orig(bid, box, out=np.full(shape, GARBAGE, dtype=np.uint32))
                rt.buffer_read = read_garbage
                stats = {}

                def keep_stats(rt=rt, close=rt.shutdown, stats=stats):
                    if rt.h is not None:
                        stats.update(rt.stats())
                    close()
                rt.shutdown = keep_stats
                res = [r[1] for r in run_program(rt, prog) if r[0] == "read"]
                if rank == 0 and stats.get("halo_fused"):
                    print("  halo copies fused into the stencil %d, incoming awaited in-kernel %d, chained rows %d"
                          % (stats["halo_fused"], stats["halo_in_waits"], stats["halo_chained"]), flush=True)
                if rank == 0 and stats.get("gather_sets"):
                    print("  all-gather sets %d, run as NCCL groups %d" % (stats["gather_sets"], stats["coll_groups"]),
                          flush=True)
            else:
                rt = cel.Runtime(world, execute=False, lookahead=mode, instr_log_path=log)
                res = []
                run_program(rt, prog)
            dist.barrier()
            mylog = [json.loads(line) for line in open(log)]
            o = OracleRuntime(world, lookahead=mode)
            run_program(o, prog)
            ok = mylog == o.log
            if args.execute:
                allres = [None] * world
                dist.all_gather_object(allres, res)
                exp = simulate(o)
                for k in range(len(res)):
                    merged = np.full_like(exp[k], GARBAGE)
                    for r in range(world):
                        a = allres[r][k]
                        merged = np.where(a != GARBAGE, a, merged)
                    defined = exp[k] != GARBAGE
                    if not np.array_equal(merged[defined], exp[k][defined]):
                        ok = False
                        if rank == 0:
                            bad = np.argwhere((merged != exp[k]) & defined)
                            print("prog %s mode %s readback %d: %d mismatches, first %s"
                                  % (prog["name"], mode, k, len(bad), bad[:3].tolist()), flush=True)
            oks = [None] * world
            dist.all_gather_object(oks, ok)
            if rank == 0:
                print("%-12s %-5s %s" % (prog["name"], mode, "ok" if all(oks) else "FAIL %s" % oks), flush=True)
            nfail += 0 if all(oks) else 1
    if rank == 0:
        print("MP_CHECK %s world=%d execute=%d" % ("PASS" if nfail == 0 else "FAIL(%d)" % nfail, world, args.execute))
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(1 if nfail else 0)


if __name__ == "__main__":
    main()
