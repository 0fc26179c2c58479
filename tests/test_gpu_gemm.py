"""The tcgen05/TMA GEMM (cvr_gemm_bf16) against a plain PyTorch fp32 reference of the same op:
C = A B^T (+ bias, ReLU) with bf16 operands, fp32 accumulation and a bf16 result."""
import pytest
import torch

pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)


@pytest.fixture(scope="module", autouse=True)
def _build():
    from paper_2605_29232_b200 import build
    build.build()


@pytest.mark.parametrize("M,N,K,bn", [(4096, 256, 1728, 64), (300, 1728, 256, 64), (1, 64, 64, 64),
                                      (4096, 1024, 1728, 128), (777, 512, 1024, 128), (129, 128, 4096, 64)])
@pytest.mark.parametrize("relu", [False, True])
@pytest.mark.parametrize("pair", [False, True])
def test_gemm_vs_fp32_reference(M, N, K, bn, relu, pair):
    from paper_2605_29232_b200 import gemm_bf16
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N + K)
    A = (torch.randn(M, K, device="cuda", generator=g) / K ** 0.25).bfloat16()
    B = (torch.randn(N, K, device="cuda", generator=g) / K ** 0.25).bfloat16()
    bias = torch.randn(N, device="cuda", generator=g) if relu else None
    C = gemm_bf16(A, B, bias=bias, bn=bn, pair=pair)
    torch.cuda.synchronize()
    ref = A.float() @ B.float().T
    if relu:
        ref = torch.relu(ref + bias)
    # bf16 output rounding (2^-9 relative) + fp32 accumulation-order differences
    err = (C.float() - ref).abs()
    tol = ref.abs() * 2 ** -8 + 1e-3
    assert torch.all(err <= tol), (err - tol).max().item()


def test_gemm_strided_operands():
    from paper_2605_29232_b200 import gemm_bf16
    A = torch.randn(256, 320, device="cuda").bfloat16()[:, :256]   # lda = 320
    B = torch.randn(128, 256, device="cuda").bfloat16()
    C = torch.zeros(256, 200, device="cuda", dtype=torch.bfloat16)[:, :128]
    gemm_bf16(A, B, C=C, bn=64)
    ref = A.float() @ B.float().T
    assert torch.all((C.float() - ref).abs() <= ref.abs() * 2 ** -8 + 1e-3)
