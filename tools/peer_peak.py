"""In-run NVLink reference: 1 GiB peer copies (cudaMemcpyPeerAsync through
torch) GPU 0 -> GPU 1, and both directions at once; CUDA events, best of 10.
Prints one JSON line (the denominator SURVEY §8(d) asks for beside 900 GB/s)."""
import json

import torch

n = 1 << 30
a = torch.empty(n, dtype=torch.uint8, device="cuda:0")
b = torch.empty(n, dtype=torch.uint8, device="cuda:1")
c = torch.empty(n, dtype=torch.uint8, device="cuda:1")
d = torch.empty(n, dtype=torch.uint8, device="cuda:0")
res = {}
for name, pairs in (("one_way_0to1", [(b, a)]), ("bidirectional", [(b, a), (d, c)])):
    best = 0.0
    for _ in range(10):
        torch.cuda.synchronize(0)
        torch.cuda.synchronize(1)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        s1 = torch.cuda.Stream(device="cuda:1")
        e0.record(torch.cuda.current_stream(0))
        with torch.cuda.device(0):
            pairs[0][0].copy_(pairs[0][1], non_blocking=True)
        if len(pairs) > 1:
            with torch.cuda.stream(s1):
                pairs[1][0].copy_(pairs[1][1], non_blocking=True)
        torch.cuda.synchronize(1)
        e1.record(torch.cuda.current_stream(0))
        torch.cuda.synchronize(0)
        ms = e0.elapsed_time(e1)
        best = max(best, n / (ms / 1e3) / 1e9)
    res[name + "_GBps_per_direction"] = best
print(json.dumps({"peer_copy_reference": res, "bytes": n, "how": "torch copy_ between devices (cudaMemcpyPeerAsync), best of 10"}))
