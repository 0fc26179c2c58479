// cvr_tile.cuh -- per-thread-row epilogue helpers shared by the tcgen05 kernels: TMEM <-> registers,
// 128-byte-swizzled bf16 staging tiles (the TMA / UMMA SWIZZLE_128B layout: 16-byte chunk c of row r
// lives at chunk c ^ (r % 8)), fp32 row I/O, and the stable sigmoid.
#pragma once
#include <cuda_bf16.h>
#include <stdint.h>

#include "cvr_ptx.cuh"

namespace cvr {
namespace tile {

__device__ __forceinline__ float sigmoid_f32(float z) {
  if (z >= 0.f) return 1.f / (1.f + expf(-z));
  const float e = expf(z);
  return e / (1.f + e);
}

// 16-byte chunk `ch` (0..7) of row `r` in a 128-B-swizzled [rows x 64] bf16 sub-tile
__device__ __forceinline__ uint32_t swz(uint32_t sub_base, int r, int ch) {
  return sub_base + r * 128 + ((ch ^ (r & 7)) << 4);
}
__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts128(uint32_t a, uint4 v) {
  asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ void ld32_tmem(uint32_t taddr, float (&v)[32]) {
  uint32_t v0[16], v1[16];
  ptx::tmem_ld_32x32b_x16(taddr, v0);
  ptx::tmem_ld_32x32b_x16(taddr + 16, v1);
  ptx::tmem_wait_ld();
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    v[j] = __uint_as_float(v0[j]);
    v[16 + j] = __uint_as_float(v1[j]);
  }
}
__device__ __forceinline__ void st32_tmem(uint32_t taddr, const float (&v)[32]) {
  uint32_t v0[16], v1[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    v0[j] = __float_as_uint(v[j]);
    v1[j] = __float_as_uint(v[16 + j]);
  }
  ptx::tmem_st_32x32b_x16(taddr, v0);
  ptx::tmem_st_32x32b_x16(taddr + 16, v1);
}
__device__ __forceinline__ void ld32_f32(const float* p, float (&v)[32]) {
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const float4 f = *reinterpret_cast<const float4*>(p + 4 * j);
    v[4 * j] = f.x;
    v[4 * j + 1] = f.y;
    v[4 * j + 2] = f.z;
    v[4 * j + 3] = f.w;
  }
}
__device__ __forceinline__ void st32_f32(float* p, const float (&v)[32]) {
#pragma unroll
  for (int j = 0; j < 8; ++j)
    *reinterpret_cast<float4*>(p + 4 * j) = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
}
// 32 columns (4 swizzled 16-byte chunks) of row r into / out of a bf16 staging sub-tile
__device__ __forceinline__ void sts32_bf16(uint32_t sub_base, int r, int ch0, const float (&v)[32]) {
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    uint4 o;
    o.x = ptx::pack_bf16(v[8 * u], v[8 * u + 1]);
    o.y = ptx::pack_bf16(v[8 * u + 2], v[8 * u + 3]);
    o.z = ptx::pack_bf16(v[8 * u + 4], v[8 * u + 5]);
    o.w = ptx::pack_bf16(v[8 * u + 6], v[8 * u + 7]);
    sts128(swz(sub_base, r, ch0 + u), o);
  }
}
__device__ __forceinline__ void lds32_bf16(uint32_t sub_base, int r, int ch0, float (&v)[32]) {
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const uint4 x = lds128(swz(sub_base, r, ch0 + u));
    const uint32_t w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      v[8 * u + 2 * j] = ptx::bf16_lo(w[j]);
      v[8 * u + 2 * j + 1] = ptx::bf16_hi(w[j]);
    }
  }
}

}  // namespace tile
}  // namespace cvr
