"""Time libcvr's tcgen05 GEMM on the config-2 shapes against cuBLAS (torch.matmul), CUDA events."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_29232_b200 import gemm_bf16

def timeit(fn, iters=20, reps=5):
    """Device time per call: `iters` calls captured in one CUDA graph (no host launch overhead)."""
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3): fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(iters): fn()
    g.replay(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): g.replay()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / (iters * reps) * 1e3

shapes = [("xV", 4096, 256, 1728), ("tU", 4096, 1728, 256), ("mlp0", 4096, 1024, 1728), ("mlp1", 4096, 512, 1024),
          ("head", 4096, 256, 512)] + ([("big", 8192, 8192, 8192)] if os.environ.get("BIG") else [])
res = []
for name, M, N, K in shapes:
    A = torch.randn(M, K, device="cuda").bfloat16(); B = torch.randn(N, K, device="cuda").bfloat16()
    C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    fl = 2 * M * N * K
    row = {"gemm": name, "M": M, "N": N, "K": K, "cublas_us": timeit(lambda: torch.matmul(A, B.T, out=C))}
    for bn in (64, 128, 192, 256):
        if N % bn == 0:
            row[f"cvr_bn{bn}_us"] = timeit(lambda: gemm_bf16(A, B, C=C, bn=bn))
    for bn in (64, 128, 256):
        if N % bn == 0:
            row[f"cvr_pair_bn{bn}_us"] = timeit(lambda: gemm_bf16(A, B, C=C, bn=bn, pair=True))
    row["cublas_tflops"] = fl / row["cublas_us"] / 1e6
    for k in list(row):
        if k.startswith("cvr_") and k.endswith("_us"):
            row[k[:-3] + "_tflops"] = fl / row[k] / 1e6
    res.append(row)
    print(json.dumps(row), flush=True)
