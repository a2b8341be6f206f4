"""Per-launch timeline of RSim rows (rank 0's device) via cel_trace_dump: rows
600-640 of W = 84,000, T = 1024, one process per GPU under torchrun."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2503_10516_b200 import cel
from workloads import programs as P
rank, world, local = bench.env_rank()
G = world
dist = None
if world > 1:
    import torch.distributed as dist
    dist.init_process_group("gloo")
torch.cuda.set_device(local)
W, T = 84000, 1024
rt = bench.make_runtime(cel, G, rank, world, dist, 4 << 30)
rt.buffer_create(2, [T, W], 4)
prog = P.rsim(W, T)
descs = [cel.task_desc(op[1]) for op in prog["ops"] if op[0] == "task"]
for d in descs[:600]: rt.submit_desc(d[0])
rt.wait()
if dist: dist.barrier()
rt.profile_enable(True)
for d in descs[600:640]: rt.submit_desc(d[0])
rt.wait()
path = "gpurun_out/trace_rsim_r%d_n%d.jsonl" % (rank, G)
rt.trace_dump(path)
if dist: dist.barrier()
rt.shutdown()
if rank == 0:
    recs = [json.loads(l) for l in open(path)]
    recs.sort(key=lambda r: r["start_us"])
    t0 = recs[0]["start_us"]
    for r in recs[-24:]:
        print("%-9s %-8s iid %6d  issued %9.1f  gpu %9.1f -> %9.1f  (%6.1f us)" % (r["kind"], r["stream"], r["iid"], r["host_issue_us"] - t0, r["start_us"] - t0, r["end_us"] - t0, r["end_us"] - r["start_us"]))
if dist: dist.destroy_process_group()
