"""Launch torch.matmul (cuBLAS) once per c2 GEMM shape so ncu can list the kernels it picks."""
import torch
for M, N, K in [(4096, 256, 1728), (4096, 1728, 256), (4096, 1024, 1728), (4096, 512, 1024), (4096, 256, 512)]:
    A = torch.randn(M, K, device="cuda").bfloat16(); B = torch.randn(N, K, device="cuda").bfloat16()
    for _ in range(3):
        C = torch.matmul(A, B.T)
    torch.cuda.synchronize()
