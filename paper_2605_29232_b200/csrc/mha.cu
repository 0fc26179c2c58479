// mha.cu -- K7: multi-head self-attention over the 64 "global tokens" of each example (config 4,
// SURVEY.md §8(a) S5', reading A20; "Transformers ... self-attention", global tokens
// PAPER.md:245), plus the finaliser of the split head (EPI_HEAD_PARTIAL).
//
//   per example b and head h (dh = 64):  O_h = softmax(Q_h K_h^T / sqrt(dh)) V_h     (S = 64 tokens)
//
// One CTA per example, 8 warps: warp w owns head w/2 and 32 query rows.  Q, K (row-major) and V^T are
// staged in padded shared memory (conflict-free fragment loads), S = Q K^T and O = P V run on the tensor
// cores as mma.sync m16n8k16 bf16 with fp32 accumulation; the 64x64 score tile of a head never leaves
// registers: row max / exp / sum in fp32 across the 4 lanes sharing a row, P rounded to bf16 as the
// second MMA's A operand (A26: P is a bf16 MMA operand).  The whole problem per (example, head) is
// 64x64x64 twice, far below a tcgen05 tile, so the legacy warp-level MMA is the right size here.
#include <cuda_bf16.h>

#include "cvr_kernels.cuh"
#include "cvr_ptx.cuh"

namespace cvr {
namespace {

constexpr int S = 64;        // tokens
constexpr int DH = 64;       // head dim
constexpr int QK_LD = 264;   // 256 + 8 bf16 padding (conflict-free: row stride = 4 banks mod 32)
constexpr int VT_LD = 72;    // 64 + 8

__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

template <int H>
__global__ void __launch_bounds__(256) mha64_kernel(const __nv_bfloat16* __restrict__ qkv, __nv_bfloat16* __restrict__ out,
                                                    int B, int out_ld) {
  constexpr int D = H * DH;           // model width (256 for 4 heads)
  extern __shared__ __align__(16) uint8_t mha_smem[];
  __nv_bfloat16* Qs = reinterpret_cast<__nv_bfloat16*>(mha_smem);
  __nv_bfloat16* Ks = Qs + S * QK_LD;
  __nv_bfloat16* Vt = Ks + S * QK_LD;   // Vt[h*64 + d][token]
  const int b = blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const __nv_bfloat16* src = qkv + (size_t)b * S * 3 * D;
  // stage Q, K row-major (16-byte loads, coalesced along the row) ...
  for (int i = tid; i < S * (2 * D / 8); i += blockDim.x) {
    const int tok = i / (2 * D / 8), c8 = (i % (2 * D / 8)) * 8;
    const uint4 v = *reinterpret_cast<const uint4*>(src + (size_t)tok * 3 * D + c8);
    if (c8 < D) *reinterpret_cast<uint4*>(&Qs[tok * QK_LD + c8]) = v;
    else *reinterpret_cast<uint4*>(&Ks[tok * QK_LD + c8 - D]) = v;
  }
  // ... and V transposed (token fastest across threads: conflict-free transposing stores)
  for (int i = tid; i < S * (D / 8); i += blockDim.x) {
    const int tok = i % S, c8 = (i / S) * 8;
    const uint4 v = *reinterpret_cast<const uint4*>(src + (size_t)tok * 3 * D + 2 * D + c8);
    const __nv_bfloat16* e = reinterpret_cast<const __nv_bfloat16*>(&v);
#pragma unroll
    for (int j = 0; j < 8; ++j) Vt[(c8 + j) * VT_LD + tok] = e[j];
  }
  __syncthreads();
  if (warp < 2 * H) {
    const int h = warp >> 1, row_base = (warp & 1) * 32;
    const int g = lane >> 2, t = lane & 3;
    const __nv_bfloat16* Q = Qs + h * DH;
    const __nv_bfloat16* Kh = Ks + h * DH;
    const __nv_bfloat16* V = Vt + h * DH * VT_LD;
    auto u32 = [](const __nv_bfloat16* p) { return *reinterpret_cast<const uint32_t*>(p); };
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      const int r0 = row_base + mt * 16;
      // ---- S = Q K^T for 16 query rows x 64 keys: 8 n-tiles x 4 k-steps
      float sc[8][4];
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) sc[nt][0] = sc[nt][1] = sc[nt][2] = sc[nt][3] = 0.f;
#pragma unroll
      for (int ks = 0; ks < DH / 16; ++ks) {
        const int k0 = ks * 16;
        uint32_t a[4];
        a[0] = u32(Q + (r0 + g) * QK_LD + k0 + 2 * t);
        a[1] = u32(Q + (r0 + g + 8) * QK_LD + k0 + 2 * t);
        a[2] = u32(Q + (r0 + g) * QK_LD + k0 + 2 * t + 8);
        a[3] = u32(Q + (r0 + g + 8) * QK_LD + k0 + 2 * t + 8);
#pragma unroll
        for (int nt = 0; nt < 8; ++nt) {
          const __nv_bfloat16* kr = Kh + (nt * 8 + g) * QK_LD + k0 + 2 * t;
          mma16816(sc[nt], a, u32(kr), u32(kr + 8));
        }
      }
      // ---- softmax over the 64 keys of rows g and g+8 (scale 1/sqrt(64) = 1/8, exact)
      float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) {
#pragma unroll
        for (int e = 0; e < 4; ++e) sc[nt][e] *= 0.125f;
        mx0 = fmaxf(mx0, fmaxf(sc[nt][0], sc[nt][1]));
        mx1 = fmaxf(mx1, fmaxf(sc[nt][2], sc[nt][3]));
      }
#pragma unroll
      for (int o = 1; o <= 2; o <<= 1) {
        mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, o));
        mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, o));
      }
      float s0 = 0.f, s1 = 0.f;
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) {
        sc[nt][0] = expf(sc[nt][0] - mx0);
        sc[nt][1] = expf(sc[nt][1] - mx0);
        sc[nt][2] = expf(sc[nt][2] - mx1);
        sc[nt][3] = expf(sc[nt][3] - mx1);
        s0 += sc[nt][0] + sc[nt][1];
        s1 += sc[nt][2] + sc[nt][3];
      }
#pragma unroll
      for (int o = 1; o <= 2; o <<= 1) {
        s0 += __shfl_xor_sync(0xffffffffu, s0, o);
        s1 += __shfl_xor_sync(0xffffffffu, s1, o);
      }
      const float i0 = 1.f / s0, i1 = 1.f / s1;
      // ---- O = P V: P (C fragments of S) re-used as A fragments; V^T gives contiguous B fragments
      float oc[8][4];
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) oc[nt][0] = oc[nt][1] = oc[nt][2] = oc[nt][3] = 0.f;
#pragma unroll
      for (int kk = 0; kk < S / 16; ++kk) {
        uint32_t a[4];
        a[0] = ptx::pack_bf16(sc[2 * kk][0] * i0, sc[2 * kk][1] * i0);
        a[1] = ptx::pack_bf16(sc[2 * kk][2] * i1, sc[2 * kk][3] * i1);
        a[2] = ptx::pack_bf16(sc[2 * kk + 1][0] * i0, sc[2 * kk + 1][1] * i0);
        a[3] = ptx::pack_bf16(sc[2 * kk + 1][2] * i1, sc[2 * kk + 1][3] * i1);
#pragma unroll
        for (int nt = 0; nt < 8; ++nt) {
          const __nv_bfloat16* vr = V + (nt * 8 + g) * VT_LD + kk * 16 + 2 * t;
          mma16816(oc[nt], a, u32(vr), u32(vr + 8));
        }
      }
      // ---- write O rows r0+g, r0+g+8, columns h*64 + nt*8 + 2t (+1)
      __nv_bfloat16* o0 = out + ((size_t)b * S + r0 + g) * out_ld + h * DH;
      __nv_bfloat16* o1 = out + ((size_t)b * S + r0 + g + 8) * out_ld + h * DH;
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) {
        *reinterpret_cast<uint32_t*>(o0 + nt * 8 + 2 * t) = ptx::pack_bf16(oc[nt][0], oc[nt][1]);
        *reinterpret_cast<uint32_t*>(o1 + nt * 8 + 2 * t) = ptx::pack_bf16(oc[nt][2], oc[nt][3]);
      }
    }
  }
}

__device__ __forceinline__ float sigmoid_f32(float z) {
  if (z >= 0.f) return 1.f / (1.f + expf(-z));
  const float e = expf(z);
  return e / (1.f + e);
}

__global__ void head_finalize_kernel(const float* __restrict__ part, int n_parts, float c, float* __restrict__ scores,
                                     int M) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= M) return;
  float z = 0.f;
  for (int j = 0; j < n_parts; ++j) z += part[(size_t)m * n_parts + j];  // fixed order: batch invariant
  scores[m] = sigmoid_f32(z + c);
}

}  // namespace

cudaError_t launch_mha64(const __nv_bfloat16* qkv, __nv_bfloat16* out, int out_ld, int B, int n_heads, cudaStream_t s) {
  if (B <= 0) return cudaSuccess;
  if (n_heads != 4) return cudaErrorInvalidValue;
  constexpr int smem = (2 * S * QK_LD + 4 * DH * VT_LD) * 2;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(mha64_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  mha64_kernel<4><<<B, 256, smem, s>>>(qkv, out, B, out_ld);
  return cudaGetLastError();
}

cudaError_t launch_head_finalize(const float* partial, int n_parts, float c, float* scores, int M, cudaStream_t s) {
  if (M <= 0) return cudaSuccess;
  head_finalize_kernel<<<(M + 255) / 256, 256, 0, s>>>(partial, n_parts, c, scores, M);
  return cudaGetLastError();
}

}  // namespace cvr
