// gemm_splitk.cu -- t = x_l V_l^T for the low-rank cross layer as a
// K-split tcgen05 GEMM over a cluster of 4 CTAs with a DSMEM reduction.
//
// Why: t is [B, r] with r = 256 and K = W = 1728.  With 128 x 64 tiles (the generic kernel) every 64-column
// MMA re-reads the 16 KB A k-block from shared memory, and TMA writes + UMMA reads of shared memory (128 B/clk
// per SM) bound the mainloop at ~5.7 us for B = 4096.  One 128 x 256 tile per row block reads A once per
// k-block (half the shared-memory bytes per FLOP), and splitting K over the 4 CTAs of a cluster keeps 4 CTAs
// per row block busy (128 CTAs at B = 4096).
//
// Per CTA (cluster rank j, row block m0):
//   mainloop   k-blocks [kb0_j, kb1_j) of the fixed partition of K (ceil(K/64/4) blocks each) -> fp32 partial
//              P_j = x_l[m0:m0+128, K_j] V[:, K_j]^T in TMEM (128 x 256), TMA ring of A (16 KB) + B (32 KB);
//   exchange   (cluster barrier: every CTA's ring is drained) the epilogue warps stage the three 64-column
//              slices owned by the peers in local shared memory, and one thread sends each to its owner with
//              a 32 KB DSMEM bulk copy (cp.async.bulk shared::cta -> shared::cluster) completing on the
//              owner's mbarrier (element-wise remote stores measured 2-3x slower);
//   reduce     CTA j waits for its 3 incoming slices, sums the 4 partials of columns [64j, 64j+64) in rank
//              order 0+1+2+3 (its own from TMEM), rounds to bf16 (t is a bf16 MMA operand, A15), stores.
// The K partition and the summation order depend on K only, never on M: every row's t is the same whatever
// batch it is in (batch invariance).
#include <cudaTypedefs.h>
#include <cuda_bf16.h>

#include "cvr_kernels.cuh"
#include "cvr_ptx.cuh"
#include "cvr_tile.cuh"

namespace cvr {
namespace {

constexpr int KS = 4;          // CTAs per cluster = K splits
constexpr int BM = 128, BK = 64, BN = 256;
constexpr int A_BYTES = BM * BK * 2;   // 16 KB
constexpr int B_BYTES = BN * BK * 2;   // 32 KB
constexpr int STAGE = A_BYTES + B_BYTES;
constexpr int STAGES = 4;
constexpr int SLOT = BM * 64 * 4;      // 32 KB: 128 rows x 64 fp32 columns, [16 float4 chunks][128 rows]
// slot k of a CTA of rank j stands for peer rank k + (k >= j) (its own rank has no slot)
constexpr int SEND = 0;                      // staging of the slices for the 3 peers: [KS-1][SLOT]
constexpr int RECV = (KS - 1) * SLOT;        // incoming slices from the 3 peers: [KS-1][SLOT]
constexpr int EPW = 4;                 // epilogue warps per TMEM lane quadrant
constexpr int NT = 32 * (2 + 4 * EPW + 1);  // A producer, MMA, 16 epilogue, B producer
constexpr int PRODUCER_B = 2 + 4 * EPW;
constexpr int SMEM = 1024 + STAGES * STAGE + 256;
static_assert(2 * (KS - 1) * SLOT <= STAGES * STAGE, "send + receive slots overlay the ring");
__device__ __forceinline__ int slot_of(int peer, int self) { return peer - (peer > self ? 1 : 0); }

// bulk copy of `bytes` from this CTA's shared memory to another CTA's (shared::cluster address), completing
// `bytes` of transaction count on the destination CTA's mbarrier (shared::cluster address)
__device__ __forceinline__ void bulk_s2c(uint32_t dst_cluster, const void* src, uint32_t bytes, uint32_t mbar_cluster) {
  asm volatile(
      "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst_cluster),
      "r"(ptx::smem_u32(src)), "r"(bytes), "r"(mbar_cluster)
      : "memory");
}

// GX (global exchange): the partial slices go through an L2-resident global scratch instead of DSMEM -- each
// epilogue warp stores its peers' slices straight from registers in a chunk-major layout (coalesced), one
// cluster barrier (release / acquire, cluster scope) orders them before the owners' loads.
// xchg layout: [row block][src rank][dst rank][16 float4 chunks][128 rows] (diagonal unused).
template <bool GX>
__global__ void __launch_bounds__(NT, 1)
    gemm_splitk_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                       __nv_bfloat16* __restrict__ out, int64_t ldo, int M, int K, float4* __restrict__ xchg,
                       unsigned long long* dbg) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE);
  uint64_t* full = bars;
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* rfull = tfull + 1;   // the 3 incoming slices have landed
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(rfull + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int j = (int)ptx::cluster_ctarank();
  const int m0 = (int)(blockIdx.x / KS) * BM;
  const int nk = K / BK, per = (nk + KS - 1) / KS;
  const int kb0 = j * per < nk ? j * per : nk, kb1 = kb0 + per < nk ? kb0 + per : nk;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&full[s], 2);
      ptx::mbar_init(&empty[s], 1);
    }
    ptx::mbar_init(tfull, 1);
    ptx::mbar_init(rfull, 1);
    ptx::fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tmA);
    ptx::prefetch_tmap(&tmB);
  }
  if (warp == 1) ptx::tmem_alloc(tmem_holder, BN);
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  if (!GX && threadIdx.x == 0) ptx::mbar_arrive_expect_tx(rfull, (KS - 1) * SLOT);
  const uint32_t tmem = *tmem_holder;
  auto stamp = [&](int i) {
    if (dbg && threadIdx.x == 2 * 32) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      dbg[blockIdx.x * 8 + i] = t;
    }
  };
  stamp(0);
  ptx::griddep_wait();
  stamp(1);
  ptx::griddep_launch();

  // ---------------------------------------------------------------- mainloop (one 128 x 256 tile)
  if (warp == 0 || warp == PRODUCER_B) {
    if (lane == 0) {
      const bool roleA = warp == 0;
      for (int kb = kb0, g = 0; kb < kb1; ++kb, ++g) {
        const int s = g % STAGES;
        if (g >= STAGES) ptx::mbar_wait(&empty[s], ((g / STAGES) - 1) & 1);
        if (roleA) {
          ptx::mbar_arrive_expect_tx(&full[s], A_BYTES);
          ptx::tma_load_2d(sA + s * A_BYTES, &tmA, &full[s], kb * BK, m0);
        } else {
          ptx::mbar_arrive_expect_tx(&full[s], B_BYTES);
          ptx::tma_load_2d(sB + s * B_BYTES, &tmB, &full[s], kb * BK, 0);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = ptx::idesc_bf16_f32(BM, BN);
      for (int kb = kb0, g = 0; kb < kb1; ++kb, ++g) {
        const int s = g % STAGES;
        ptx::mbar_wait(&full[s], (g / STAGES) & 1);
        ptx::tc_fence_after();
        const uint64_t ad = ptx::sdesc_kmajor_sw128(ptx::smem_u32(sA + s * A_BYTES));
        const uint64_t bd = ptx::sdesc_kmajor_sw128(ptx::smem_u32(sB + s * B_BYTES));
#pragma unroll
        for (int k = 0; k < BK / 16; ++k) ptx::umma_bf16_ss(tmem, ad + 2 * k, bd + 2 * k, idesc, (g | k) != 0);
        ptx::umma_commit(&empty[s]);
      }
      ptx::umma_commit(tfull);
    }
  } else {
    ptx::mbar_wait(tfull, 0);  // this CTA's partial is complete (and its ring no longer read)
    stamp(3);
  }
  const bool epi = warp >= 2 && warp < PRODUCER_B;
  const int q = warp & 3, part = (warp - 2) >> 2, r = q * 32 + lane;
  const int64_t rb = blockIdx.x / KS;
  if constexpr (GX) {
    // ---------------------------------------------------------------- exchange through L2
    if (epi && part != j) {
      float4* dst = xchg + ((rb * KS + j) * KS + part) * (16 * BM);
      const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16) + part * 64;
#pragma unroll
      for (int c = 0; c < 64; c += 32) {
        float v[32];
        tile::ld32_tmem(trow + c, v);
#pragma unroll
        for (int u = 0; u < 8; ++u)
          __stcg(dst + ((c >> 2) + u) * BM + r, make_float4(v[4 * u], v[4 * u + 1], v[4 * u + 2], v[4 * u + 3]));
      }
    }
    stamp(2);
    ptx::tc_fence_before();
    ptx::cluster_sync();  // release / acquire at cluster scope: every peer's slices are in L2
    ptx::tc_fence_after();
    stamp(5);
  } else {
  ptx::tc_fence_before();
  ptx::cluster_sync();  // every CTA of the cluster has drained its ring: receive slots may be written
  ptx::tc_fence_after();
  stamp(4);

  // ---------------------------------------------------------------- exchange: partial columns -> owners
  if (epi && part != j) {
    // columns [64 part, 64 part + 64) of rows 32q..32q+31 belong to CTA `part`: stage them in send slot part
    const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16) + part * 64;
    uint8_t* dst = smem + SEND + slot_of(part, j) * SLOT;
#pragma unroll
    for (int c = 0; c < 64; c += 32) {
      float v[32];
      tile::ld32_tmem(trow + c, v);
#pragma unroll
      for (int u = 0; u < 8; ++u)
        *reinterpret_cast<float4*>(dst + (((c >> 2) + u) * BM + r) * 16) =
            make_float4(v[4 * u], v[4 * u + 1], v[4 * u + 2], v[4 * u + 3]);
    }
    ptx::fence_async_smem();  // generic-proxy writes -> visible to the bulk copy (async proxy)
  }
  if (epi) ptx::named_bar_sync(1, 32 * 4 * EPW);
  if (warp == 2 && lane == 0) {
    for (int p = 0; p < KS; ++p) {
      if (p == j) continue;
      bulk_s2c(ptx::mapa(smem + RECV + slot_of(j, p) * SLOT, (uint32_t)p), smem + SEND + slot_of(p, j) * SLOT, SLOT,
               ptx::mapa(rfull, (uint32_t)p));
    }
    ptx::bulk_commit();
  }
  stamp(2);
  if (epi) ptx::mbar_wait_cluster(rfull, 0);  // the peers' slices for our columns have landed
  stamp(5);
  }

  // ---------------------------------------------------------------- reduce own 64 columns, bf16 out
  if (epi) {
    // warp (q, part): rows 32q.., columns 64j + 16 part .. +16 (4 float4 chunks)
    const int m = m0 + r;
    float4 own[4];  // this CTA's partial of columns 64j + 16 part .. +16, straight from TMEM
    {
      uint32_t v[16];
      ptx::tmem_ld_32x32b_x16(tmem + ((uint32_t)(q * 32) << 16) + j * 64 + part * 16, v);
      ptx::tmem_wait_ld();
#pragma unroll
      for (int u = 0; u < 4; ++u)
        own[u] = make_float4(__uint_as_float(v[4 * u]), __uint_as_float(v[4 * u + 1]), __uint_as_float(v[4 * u + 2]),
                             __uint_as_float(v[4 * u + 3]));
    }
    if (m < M) {
      float s[16];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int ch = part * 4 + u;
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int src = 0; src < KS; ++src) {  // fixed order 0 + 1 + 2 + 3 (the first add is exact)
          float4 p;
          if (src == j) p = own[u];
          else if constexpr (GX) p = __ldcg(xchg + ((rb * KS + src) * KS + j) * (16 * BM) + ch * BM + r);
          else p = *reinterpret_cast<const float4*>(smem + RECV + slot_of(src, j) * SLOT + (ch * BM + r) * 16);
          acc.x += p.x;
          acc.y += p.y;
          acc.z += p.z;
          acc.w += p.w;
        }
        s[4 * u] = acc.x;
        s[4 * u + 1] = acc.y;
        s[4 * u + 2] = acc.z;
        s[4 * u + 3] = acc.w;
      }
      uint4 o0, o1;
      o0.x = ptx::pack_bf16(s[0], s[1]);
      o0.y = ptx::pack_bf16(s[2], s[3]);
      o0.z = ptx::pack_bf16(s[4], s[5]);
      o0.w = ptx::pack_bf16(s[6], s[7]);
      o1.x = ptx::pack_bf16(s[8], s[9]);
      o1.y = ptx::pack_bf16(s[10], s[11]);
      o1.z = ptx::pack_bf16(s[12], s[13]);
      o1.w = ptx::pack_bf16(s[14], s[15]);
      uint4* op = reinterpret_cast<uint4*>(out + (int64_t)m * ldo + j * 64 + part * 16);
      op[0] = o0;
      op[1] = o1;
    }
  }
  stamp(6);
  if (!GX && warp == 2 && lane == 0) ptx::bulk_wait_read<0>();  // our outgoing slices have been read
  __syncthreads();
  if (warp == 1) ptx::tmem_dealloc(tmem, BN);
}

}  // namespace

cudaError_t launch_gemm_splitk(const GemmArgs& g, cudaStream_t s) {
  if (g.M <= 0) return cudaSuccess;
  if (g.N != BN || g.K % BK || g.K / BK < KS || !g.out_bf16 || g.ld_x < BN) return cudaErrorInvalidValue;
  static bool attr_done = false;
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(gemm_splitk_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(gemm_splitk_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    if (e != cudaSuccess) return e;
    attr_done = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(((g.M + BM - 1) / BM) * KS);
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = SMEM;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = g.pdl ? 1 : 0;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = KS;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  float4* xchg = reinterpret_cast<float4*>(g.partial);  // non-null: exchange through L2 (GX)
  if (xchg)
    return cudaLaunchKernelEx(&cfg, gemm_splitk_kernel<true>, *g.tmA, *g.tmB, g.out_bf16, g.ld_x, g.M, g.K, xchg, g.dbg);
  return cudaLaunchKernelEx(&cfg, gemm_splitk_kernel<false>, *g.tmA, *g.tmB, g.out_bf16, g.ld_x, g.M, g.K, xchg, g.dbg);
}

}  // namespace cvr
