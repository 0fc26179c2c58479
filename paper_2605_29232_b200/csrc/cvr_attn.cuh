// cvr_attn.cuh -- the per-warp core of config 4's 64-token attention (SURVEY.md §8(a) S5', reading A20),
// shared by mha64 (mha.cu) and the fused QKV-projection + attention GEMM epilogue (gemm_tc.cu, EPI_ATTN) so the
// two produce bit-identical O.  One warp computes 16 query rows of one (example, head):
//   S = Q K^T / 8 (mma.sync m16n8k16, bf16 operands, fp32 accumulate), row softmax in fp32 across the 4 lanes
//   sharing a row, P rounded to bf16 (A26), O = P V -- then writes its 16 rows of O (bf16) over its own Q rows.
// Q, K, V: 64 x 64 bf16 in shared memory with row stride LD elements (LD = 72: conflict-free ldmatrix).
#pragma once
#include <cuda_bf16.h>
#include <stdint.h>

#include "cvr_ptx.cuh"

namespace cvr {
namespace attn {

__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(ptx::smem_u32(p)));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(ptx::smem_u32(p)));
}

template <int LD>
__device__ __forceinline__ void rows16(__nv_bfloat16* Qs, const __nv_bfloat16* Ks, const __nv_bfloat16* Vs, int r0,
                                       int lane) {
  const int g = lane >> 2, t = lane & 3;
  // ---- S = Q K^T (16 rows x 64 keys)
  float sc[8][4];
#pragma unroll
  for (int nt = 0; nt < 8; ++nt) sc[nt][0] = sc[nt][1] = sc[nt][2] = sc[nt][3] = 0.f;
#pragma unroll
  for (int ks = 0; ks < 4; ++ks) {
    uint32_t a[4];
    ldsm_x4(a, Qs + (r0 + (lane & 7) + ((lane >> 3) & 1) * 8) * LD + ks * 16 + (lane >> 4) * 8);
#pragma unroll
    for (int np = 0; np < 4; ++np) {  // two 8-key n-tiles per ldmatrix.x4
      uint32_t bq[4];
      ldsm_x4(bq, Ks + (np * 16 + (lane & 7) + (lane >> 4) * 8) * LD + ks * 16 + ((lane >> 3) & 1) * 8);
      mma16816(sc[2 * np], a, bq[0], bq[1]);
      mma16816(sc[2 * np + 1], a, bq[2], bq[3]);
    }
  }
  // ---- softmax over 64 keys for rows g and g+8 (scale 1/8 exact), fp32
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
  // ---- O = P V (P re-used from the S fragments as bf16 A operands; V via ldmatrix.trans)
  float oc[8][4];
#pragma unroll
  for (int nt = 0; nt < 8; ++nt) oc[nt][0] = oc[nt][1] = oc[nt][2] = oc[nt][3] = 0.f;
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) {
    uint32_t a[4];
    a[0] = ptx::pack_bf16(sc[2 * kk][0] * i0, sc[2 * kk][1] * i0);
    a[1] = ptx::pack_bf16(sc[2 * kk][2] * i1, sc[2 * kk][3] * i1);
    a[2] = ptx::pack_bf16(sc[2 * kk + 1][0] * i0, sc[2 * kk + 1][1] * i0);
    a[3] = ptx::pack_bf16(sc[2 * kk + 1][2] * i1, sc[2 * kk + 1][3] * i1);
#pragma unroll
    for (int np = 0; np < 4; ++np) {  // two 8-wide dh tiles per ldmatrix.x4.trans
      uint32_t bv[4];
      ldsm_x4_t(bv, Vs + (kk * 16 + (lane & 7) + ((lane >> 3) & 1) * 8) * LD + np * 16 + (lane >> 4) * 8);
      mma16816(oc[2 * np], a, bv[0], bv[1]);
      mma16816(oc[2 * np + 1], a, bv[2], bv[3]);
    }
  }
  // ---- O over this warp's own 16 rows of Qs (the caller stores them)
  __nv_bfloat16* Os = Qs + r0 * LD;
#pragma unroll
  for (int nt = 0; nt < 8; ++nt) {
    *reinterpret_cast<uint32_t*>(Os + g * LD + nt * 8 + 2 * t) = ptx::pack_bf16(oc[nt][0], oc[nt][1]);
    *reinterpret_cast<uint32_t*>(Os + (g + 8) * LD + nt * 8 + 2 * t) = ptx::pack_bf16(oc[nt][2], oc[nt][3]);
  }
}

}  // namespace attn
}  // namespace cvr
