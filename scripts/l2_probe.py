"""Effective copy bandwidth vs working-set size (L2-resident vs HBM), CUDA-graph timed."""
import torch
def bw(nbytes, iters=50):
    n = nbytes // 2
    x = torch.randn(n, device="cuda").bfloat16(); y = torch.empty_like(x)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3): y.copy_(x)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(iters): y.copy_(x)
    g.replay(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); g.replay(); b.record(); torch.cuda.synchronize()
    t = a.elapsed_time(b) / iters / 1e3
    return 2 * nbytes / t / 1e12, t * 1e6
for mb in (2, 8, 16, 32, 48, 64, 128, 512, 2048):
    tb, us = bw(mb << 20)
    print(f"copy {mb:5d} MB x2 (r+w): {tb:6.2f} TB/s  {us:8.2f} us")
