"""Pinned host -> device copy bandwidth on this box (what bounds the host-fed e2e number): one copy of the c2
per-batch input size and larger, back to back on one stream, CUDA events."""
import json
import torch

dev = torch.device("cuda")
s = torch.cuda.Stream()
for mb in (0.5, 3.18, 16, 64, 256):
    n = int(mb * 2**20)
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    for _ in range(3):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    reps = max(5, int(2e9 / n))
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        a.record(s)
        for _ in range(reps):
            d.copy_(h, non_blocking=True)
        b.record(s)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    print(json.dumps({"MB": mb, "us_per_copy": round(ms * 1e3, 1), "GBps": round(n / ms / 1e6, 1)}))
# device -> host
n = 64 * 2**20
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device=dev)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(10):
    h.copy_(d, non_blocking=True)
b.record()
torch.cuda.synchronize()
print(json.dumps({"D2H_MB": 64, "GBps": round(n * 10 / a.elapsed_time(b) / 1e6, 1)}))
import os
print(json.dumps({"numa_nodes": sorted(os.listdir("/sys/devices/system/node")) if os.path.exists("/sys/devices/system/node") else None,
                  "cpu_affinity": len(os.sched_getaffinity(0))}))
