"""cuBLAS (torch.matmul, bf16 in / fp32 accumulate) on config 2's dense-stage GEMM shapes, back to back on one
stream with CUDA events: a library reference point for the per-role chain times of bench.py (not on any hot path)."""
import json
import torch

B = 4096
shapes = {"xV": (B, 1728, 256), "U (plain store)": (B, 256, 1728), "mlp1": (B, 1728, 1024), "mlp2": (B, 1024, 512),
          "mlp3": (B, 512, 256)}
for name, (M, K, N) in shapes.items():
    a = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(N, K, device="cuda", dtype=torch.bfloat16)
    c = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    for _ in range(20):
        torch.matmul(a, b.t(), out=c)
    torch.cuda.synchronize()
    reps = 200
    g = torch.cuda.CUDAGraph()  # one graph of `reps` GEMMs: device time, not the host's launch rate
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        torch.matmul(a, b.t(), out=c)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                torch.matmul(a, b.t(), out=c)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / reps * 1e3
    print(json.dumps({"gemm": name, "M": M, "K": K, "N": N, "us": round(us, 2),
                      "tflops": round(2 * M * N * K / us / 1e6, 1)}))
