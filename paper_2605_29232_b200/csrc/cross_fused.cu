// cross_fused.cu -- K5: one low-rank DCN-v2 cross layer in ONE kernel:
//
//     t       = x_l V_l^T                      (V_l [r, W], r = 256)
//     x_{l+1} = x0 * (t U_l^T + b_l) + x_l     (U_l [W, r], bias per A9)
//
// A cluster of 4 CTAs owns one 128-row block:
//   phase A  CTA j computes a K-split partial of t over k-blocks [j*ceil(nk/4), ...) with a
//            128 x 256 tcgen05 MMA (N = r = 256: 48 KB of operands per 64-deep k-block, half the
//            bytes/FLOP of a 128 x 64 tile) into TMEM, and writes the fp32 partial to an L2-resident
//            scratch buffer (coalesced [chunk][row][4] layout);
//   cluster barrier;
//   phase B  CTA j sums the 4 partials of its 64 columns in the fixed order 0+1+2+3 (deterministic and
//            independent of the batch size: batch invariance), rounds to bf16 (A15:
//            t is a bf16 MMA operand) and writes its slice of t;
//   cluster barrier;
//   phase C  every CTA TMA-loads the whole t block (128 x 256 bf16, 64 KB) ONCE into shared memory and
//            streams its quarter of the U_l tiles (64 columns each) through a 2-deep ring; each tile is
//            one 128 x 64 x 256 MMA into one of two TMEM accumulators, and the epilogue warps apply
//            x0 * (acc + b) + x_l with x0 / x_l tiles loaded by TMA, writing x_{l+1} by TMA store.
// Compared with two GEMM launches this removes one launch + pipeline fill and the 27-fold re-read of t
// by the U GEMM's N tiles.
#include <cudaTypedefs.h>
#include <cuda_bf16.h>

#include "cvr_kernels.cuh"
#include "cvr_ptx.cuh"

namespace cvr {
namespace {

constexpr int CL = 4;      // CTAs per cluster (per 128-row block)
constexpr int BM = 128;
constexpr int BK = 64;
constexpr int BN = 64;     // phase-C tile width
constexpr int R = 256;     // cross rank
constexpr int kThreads = 192;
constexpr int KB = 1024;

// shared memory map (phase A and phase C overlay the same bytes)
constexpr int A_BYTES = BM * BK * 2;           // 16 KB
constexpr int VB_BYTES = R * BK * 2;           // 32 KB
constexpr int STAGE_A = A_BYTES + VB_BYTES;    // 48 KB
constexpr int STAGES_A = 4;                    // 192 KB
constexpr int SUB = BM * 64 * 2;               // 16 KB: a 128 x 64 bf16 swizzled sub-tile
constexpr int TB_OFF = 0;                      // t block: R/64 sub-tiles (64 KB)
constexpr int UB_OFF = 64 * KB;                // U ring: 2 x (R/64 x [64 x 64]) (64 KB)
constexpr int UTILE = (R / 64) * BN * 128;     // 32 KB
constexpr int EIN_OFF = 128 * KB;              // x0 + x_l tiles: 2 x 32 KB
constexpr int OUT_OFF = 192 * KB;              // out tiles: 2 x 16 KB
constexpr int DATA_BYTES = 224 * KB;
constexpr int SMEM = 1024 + DATA_BYTES + 256;
static_assert(STAGES_A * STAGE_A <= DATA_BYTES, "phase A ring");
constexpr int TMEM_COLS = 512;                 // [0,256) phase-A accumulator, [256,384) phase C x2

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

__global__ void __launch_bounds__(kThreads, 1)
    cross_fused_kernel(const __grid_constant__ CUtensorMap tmXl,   // x_l [M, W] box {64,128} (A of phase A, epilogue x_l)
                       const __grid_constant__ CUtensorMap tmV,    // V [R, W]  box {64,256}
                       const __grid_constant__ CUtensorMap tmT,    // t [M, R]  box {64,128}
                       const __grid_constant__ CUtensorMap tmU,    // U [W, R]  box {64,64}
                       const __grid_constant__ CUtensorMap tmX0,   // x0 [M, W] box {64,128}
                       const __grid_constant__ CUtensorMap tmOut,  // x_{l+1} [M, W] box {64,32}
                       const float* __restrict__ bias, float* __restrict__ part, __nv_bfloat16* __restrict__ t_out,
                       int M, int W, unsigned long long* __restrict__ dbg) {
#define CF_STAMP(i)                                                                              \
  if (dbg && threadIdx.x == 64) {                                                                \
    unsigned long long t_;                                                                       \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                      \
    dbg[blockIdx.x * 8 + (i)] = t_;                                                              \
  }
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + DATA_BYTES);
  uint64_t* fullA = bars;                 // [4]
  uint64_t* emptyA = fullA + STAGES_A;    // [4]
  uint64_t* tfullA = emptyA + STAGES_A;   // [1]
  uint64_t* tload = tfullA + 1;           // [1]
  uint64_t* ufull = tload + 1;            // [2]
  uint64_t* uempty = ufull + 2;           // [2]
  uint64_t* tfull = uempty + 2;           // [2]
  uint64_t* tempty = tfull + 2;           // [2] (4 epilogue warps)
  uint64_t* efull = tempty + 2;           // [2]
  uint64_t* eempty = efull + 2;           // [2] (4 epilogue warps)
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(eempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int j = (int)ptx::cluster_ctarank();     // == blockIdx.x % CL
  const int mb = blockIdx.x / CL, nmb = gridDim.x / CL;
  const int m0 = mb * BM;
  const int nk = W / BK;
  const int per = (nk + CL - 1) / CL;
  const int kb0 = j * per, kb1 = min(nk, kb0 + per);
  const int n_nt = W / BN;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES_A; ++s) {
      ptx::mbar_init(&fullA[s], 1);
      ptx::mbar_init(&emptyA[s], 1);
    }
    ptx::mbar_init(tfullA, 1);
    ptx::mbar_init(tload, 1);
    for (int a = 0; a < 2; ++a) {
      ptx::mbar_init(&ufull[a], 1);
      ptx::mbar_init(&uempty[a], 1);
      ptx::mbar_init(&tfull[a], 1);
      ptx::mbar_init(&tempty[a], 4);
      ptx::mbar_init(&efull[a], 1);
      ptx::mbar_init(&eempty[a], 4);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tmXl);
    ptx::prefetch_tmap(&tmV);
    ptx::prefetch_tmap(&tmT);
    ptx::prefetch_tmap(&tmU);
    ptx::prefetch_tmap(&tmX0);
    ptx::prefetch_tmap(&tmOut);
  }
  if (warp == 1) ptx::tmem_alloc(tmem_holder, TMEM_COLS);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  CF_STAMP(0);
  ptx::griddep_wait();
  CF_STAMP(1);

  // ============================ phase A: K-split partial of t = x_l V^T ============================
  if (warp == 0) {
    if (lane == 0) {
      for (int kb = kb0, g = 0; kb < kb1; ++kb, ++g) {
        const int s = g % STAGES_A;
        if (g >= STAGES_A) ptx::mbar_wait(&emptyA[s], ((g / STAGES_A) - 1) & 1);
        ptx::mbar_arrive_expect_tx(&fullA[s], STAGE_A);
        uint8_t* st = smem + s * STAGE_A;
        ptx::tma_load_2d(st, &tmXl, &fullA[s], kb * BK, m0);
        ptx::tma_load_2d(st + A_BYTES, &tmV, &fullA[s], kb * BK, 0);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = ptx::idesc_bf16_f32(BM, R);
      for (int kb = kb0, g = 0; kb < kb1; ++kb, ++g) {
        const int s = g % STAGES_A;
        ptx::mbar_wait(&fullA[s], (g / STAGES_A) & 1);
        ptx::tc_fence_after();
        uint8_t* st = smem + s * STAGE_A;
        const uint64_t ad = ptx::sdesc_kmajor_sw128(ptx::smem_u32(st));
        const uint64_t bd = ptx::sdesc_kmajor_sw128(ptx::smem_u32(st + A_BYTES));
#pragma unroll
        for (int k = 0; k < BK / 16; ++k) ptx::umma_bf16_ss(tmem, ad + 2 * k, bd + 2 * k, idesc, (g | k) != 0);
        ptx::umma_commit(&emptyA[s]);
      }
      ptx::umma_commit(tfullA);
    }
    __syncwarp();
  } else {
    const int q = warp & 3, r = q * 32 + lane;
    ptx::mbar_wait(tfullA, 0);
    ptx::tc_fence_after();
    const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16);
    // partial layout: part[((j * nmb + mb) * (R/4) + chunk) * 128 + r] (float4), coalesced per warp
    float4* pp = reinterpret_cast<float4*>(part) + ((size_t)(j * nmb + mb) * (R / 4)) * 128 + r;
#pragma unroll 1
    for (int c = 0; c < R; c += 32) {
      uint32_t v0[16], v1[16];
      ptx::tmem_ld_32x32b_x16(trow + c, v0);
      ptx::tmem_ld_32x32b_x16(trow + c + 16, v1);
      ptx::tmem_wait_ld();
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        pp[(size_t)(c / 4 + u) * 128] = make_float4(__uint_as_float(v0[4 * u]), __uint_as_float(v0[4 * u + 1]),
                                                    __uint_as_float(v0[4 * u + 2]), __uint_as_float(v0[4 * u + 3]));
        pp[(size_t)(c / 4 + 4 + u) * 128] = make_float4(__uint_as_float(v1[4 * u]), __uint_as_float(v1[4 * u + 1]),
                                                        __uint_as_float(v1[4 * u + 2]), __uint_as_float(v1[4 * u + 3]));
      }
    }
  }
  CF_STAMP(2);
  ptx::tc_fence_before();
  ptx::cluster_sync();
  CF_STAMP(3);

  // ============================ phase B: fixed-order reduction of this CTA's 64 columns ============
  if (warp >= 2) {
    const int q = warp & 3, r = q * 32 + lane;
    const float4* p0 = reinterpret_cast<const float4*>(part);
    const size_t split_stride = (size_t)nmb * (R / 4) * 128;
    const size_t base = ((size_t)mb * (R / 4) + j * 16) * 128 + r;
    const bool live = m0 + r < M;
#pragma unroll 2
    for (int ch = 0; ch < 16; ch += 2) {
      float s[8];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        float4 acc = p0[base + (size_t)(ch + h) * 128];
#pragma unroll
        for (int sp = 1; sp < CL; ++sp) {
          const float4 v = p0[base + sp * split_stride + (size_t)(ch + h) * 128];
          acc.x += v.x;
          acc.y += v.y;
          acc.z += v.z;
          acc.w += v.w;
        }
        s[4 * h] = acc.x;
        s[4 * h + 1] = acc.y;
        s[4 * h + 2] = acc.z;
        s[4 * h + 3] = acc.w;
      }
      if (live) {
        uint4 o;
        o.x = ptx::pack_bf16(s[0], s[1]);
        o.y = ptx::pack_bf16(s[2], s[3]);
        o.z = ptx::pack_bf16(s[4], s[5]);
        o.w = ptx::pack_bf16(s[6], s[7]);
        *reinterpret_cast<uint4*>(t_out + (size_t)(m0 + r) * R + j * 64 + ch * 4) = o;
      }
    }
    ptx::fence_async_global();  // these generic stores are read by TMA (async proxy) after the barrier
  }
  CF_STAMP(4);
  ptx::cluster_sync();
  CF_STAMP(5);

  // ============================ phase C: x_{l+1} = x0 * (t U^T + b) + x_l ============================
  uint8_t* TB = smem + TB_OFF;
  uint8_t* UB = smem + UB_OFF;
  uint8_t* EIN = smem + EIN_OFF;
  uint8_t* OUT = smem + OUT_OFF;
  if (warp == 0) {
    if (lane == 0) {
      ptx::mbar_arrive_expect_tx(tload, R / 64 * SUB);
#pragma unroll
      for (int s = 0; s < R / 64; ++s) ptx::tma_load_2d(TB + s * SUB, &tmT, tload, s * 64, m0);
      int it = 0;
      for (int nt = j; nt < n_nt; nt += CL, ++it) {
        const int a = it & 1, n0 = nt * BN;
        if (it >= 2) ptx::mbar_wait(&eempty[a], ((it >> 1) - 1) & 1);
        ptx::mbar_arrive_expect_tx(&efull[a], 2 * SUB);
        ptx::tma_load_2d(EIN + a * 2 * SUB, &tmX0, &efull[a], n0, m0);
        ptx::tma_load_2d(EIN + a * 2 * SUB + SUB, &tmXl, &efull[a], n0, m0);
        if (it >= 2) ptx::mbar_wait(&uempty[a], ((it >> 1) - 1) & 1);
        ptx::mbar_arrive_expect_tx(&ufull[a], UTILE);
#pragma unroll
        for (int s = 0; s < R / 64; ++s) ptx::tma_load_2d(UB + a * UTILE + s * (BN * 128), &tmU, &ufull[a], s * 64, n0);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = ptx::idesc_bf16_f32(BM, BN);
      ptx::mbar_wait(tload, 0);
      int it = 0;
      for (int nt = j; nt < n_nt; nt += CL, ++it) {
        const int a = it & 1;
        if (it >= 2) ptx::mbar_wait(&tempty[a], ((it >> 1) - 1) & 1);
        ptx::mbar_wait(&ufull[a], (it >> 1) & 1);
        ptx::tc_fence_after();
        const uint32_t acc = tmem + R + a * BN;
#pragma unroll
        for (int s = 0; s < R / 64; ++s) {
          const uint64_t ad = ptx::sdesc_kmajor_sw128(ptx::smem_u32(TB + s * SUB));
          const uint64_t bd = ptx::sdesc_kmajor_sw128(ptx::smem_u32(UB + a * UTILE + s * (BN * 128)));
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) ptx::umma_bf16_ss(acc, ad + 2 * k, bd + 2 * k, idesc, (s | k) != 0);
        }
        ptx::umma_commit(&uempty[a]);
        ptx::umma_commit(&tfull[a]);
      }
    }
    __syncwarp();
  } else {
    const int q = warp & 3, r = q * 32 + lane;
    int it = 0;
    for (int nt = j; nt < n_nt; nt += CL, ++it) {
      const int a = it & 1, n0 = nt * BN;
      ptx::mbar_wait(&tfull[a], (it >> 1) & 1);
      ptx::tc_fence_after();
      ptx::mbar_wait(&efull[a], (it >> 1) & 1);
      if (lane == 0) ptx::bulk_wait_read<1>();
      __syncwarp();
      const uint32_t trow = tmem + R + a * BN + ((uint32_t)(q * 32) << 16);
      const uint32_t x0b = ptx::smem_u32(EIN + a * 2 * SUB), xlb = x0b + SUB;
      const uint32_t ob = ptx::smem_u32(OUT + a * SUB);
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        uint32_t v0[16], v1[16];
        ptx::tmem_ld_32x32b_x16(trow + c, v0);
        ptx::tmem_ld_32x32b_x16(trow + c + 16, v1);
        ptx::tmem_wait_ld();
        float v[32];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          v[i] = __uint_as_float(v0[i]);
          v[16 + i] = __uint_as_float(v1[i]);
        }
        const int ch0 = c >> 3;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          float* w = v + 8 * u;
          const uint4 xa = lds128(swz(x0b, r, ch0 + u));
          const uint4 xb = lds128(swz(xlb, r, ch0 + u));
          const uint32_t x0w[4] = {xa.x, xa.y, xa.z, xa.w}, xlw[4] = {xb.x, xb.y, xb.z, xb.w};
          const int n = n0 + c + 8 * u;
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            w[2 * i] = ptx::bf16_lo(x0w[i]) * (w[2 * i] + __ldg(bias + n + 2 * i)) + ptx::bf16_lo(xlw[i]);
            w[2 * i + 1] = ptx::bf16_hi(x0w[i]) * (w[2 * i + 1] + __ldg(bias + n + 2 * i + 1)) + ptx::bf16_hi(xlw[i]);
          }
          uint4 o;
          o.x = ptx::pack_bf16(w[0], w[1]);
          o.y = ptx::pack_bf16(w[2], w[3]);
          o.z = ptx::pack_bf16(w[4], w[5]);
          o.w = ptx::pack_bf16(w[6], w[7]);
          sts128(swz(ob, r, ch0 + u), o);
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        ptx::mbar_arrive(&tempty[a]);
        ptx::mbar_arrive(&eempty[a]);
      }
      ptx::fence_async_smem();
      __syncwarp();
      if (lane == 0) {
        ptx::tma_store_2d(&tmOut, OUT + a * SUB + q * 32 * 128, n0, m0 + q * 32);
        ptx::bulk_commit();
      }
    }
    if (lane == 0) ptx::bulk_wait<0>();
  }
  CF_STAMP(6);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::griddep_launch();
  if (warp == 1) ptx::tmem_dealloc(tmem, TMEM_COLS);
}

}  // namespace

size_t cross_fused_partial_bytes(int max_batch) {
  const size_t mblocks = (size_t)(max_batch + BM - 1) / BM;
  return (size_t)CL * mblocks * BM * R * sizeof(float);
}

cudaError_t launch_cross_fused(const CrossFusedArgs& g, cudaStream_t s) {
  if (g.M <= 0) return cudaSuccess;
  if (g.R != R || g.W % BN || g.W / BK < CL) return cudaErrorInvalidValue;
  static bool attr_done = false;
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(cross_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    if (e != cudaSuccess) return e;
    attr_done = true;
  }
  const int mblocks = (g.M + BM - 1) / BM;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(mblocks * CL);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = SMEM;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = g.pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, cross_fused_kernel, *g.tmXl, *g.tmV, *g.tmT, *g.tmU, *g.tmX0, *g.tmOut, g.bias,
                            g.part, g.t_out, g.M, g.W, g.dbg);
}

}  // namespace cvr
