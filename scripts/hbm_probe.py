import torch, time
n = 1 << 30
a = torch.empty(n, dtype=torch.bfloat16, device="cuda").normal_(); b = torch.empty_like(a)
best = 1e9
for i in range(10):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); s.record(); b.copy_(a); e.record(); torch.cuda.synchronize()
    best = min(best, s.elapsed_time(e))
print("copy 1Gi bf16 best ms", best, "GB/s r+w", 2 * 2 * n / best / 1e6)
# read-only: sum
best = 1e9
for i in range(5):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); s.record(); x = a.view(torch.int32).sum(dtype=torch.int64); e.record(); torch.cuda.synchronize()
    best = min(best, s.elapsed_time(e))
print("sum read GB/s", 2 * n / best / 1e6)
import subprocess
print(subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.mem,clocks.max.mem,power.draw", "--format=csv"], capture_output=True, text=True).stdout)
