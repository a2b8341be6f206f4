"""Per-launch timeline of WaveSim steps (rank 0's device) via cel_trace_dump;
prints a per-step breakdown. Run under torchrun for N>1."""
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
n = 16384
rt = bench.make_runtime(cel, G, rank, world, dist, int(2 * (n // G + 2) * n * 4 * 1.05) + (512 << 20))
rt.buffer_create(2, [n, n], 4); rt.buffer_create(2, [n, n], 4)
for op in P.wavesim_init(n): rt.task_submit(op[1])
d = [cel.task_desc(P.wavesim_step(n, k)[1]) for k in (0, 1)]
for k in range(100): rt.submit_desc(d[k % 2][0])
rt.wait()
if dist: dist.barrier()
rt.profile_enable(True)
for k in range(100, 140): rt.submit_desc(d[k % 2][0])
rt.wait()
path = "gpurun_out/trace_r%d_n%d.jsonl" % (rank, G)
os.makedirs("gpurun_out", exist_ok=True)
rt.trace_dump(path)
if dist: dist.barrier()
rt.shutdown()
if rank == 0:
    recs = [json.loads(l) for l in open(path)]
    recs.sort(key=lambda r: r["start_us"])
    t0 = recs[0]["start_us"]
    for r in recs[-24:]:
        print("%-6s %-8s iid %6d  issued %9.1f  gpu %9.1f -> %9.1f  (%6.1f us)" % (r["kind"], r["stream"], r["iid"], r["host_issue_us"] - t0, r["start_us"] - t0, r["end_us"] - t0, r["end_us"] - r["start_us"]))
if dist: dist.destroy_process_group()
