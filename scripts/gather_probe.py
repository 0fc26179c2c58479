"""Random row-gather bandwidth (torch index_select) vs row size, uniform over a table larger than L2."""
import torch
def run(row_bytes, table_gb=2.0, n=1 << 21, iters=20):
    d = row_bytes // 2
    rows = int(table_gb * 1e9 / row_bytes)
    T = torch.empty(rows, d, dtype=torch.bfloat16, device="cuda").normal_()
    idx = torch.randint(0, rows, (n,), device="cuda")
    out = torch.empty(n, d, dtype=torch.bfloat16, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        torch.index_select(T, 0, idx, out=out)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(iters): torch.index_select(T, 0, idx, out=out)
    g.replay(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); g.replay(); b.record(); torch.cuda.synchronize()
    t = a.elapsed_time(b) / iters / 1e3
    print(f"row {row_bytes:4d} B: gather read {n*row_bytes/t/1e12:.2f} TB/s, read+write {2*n*row_bytes/t/1e12:.2f} TB/s, {t*1e6:.1f} us")
    del T
for rb in (64, 128, 256, 512, 1024):
    run(rb)
