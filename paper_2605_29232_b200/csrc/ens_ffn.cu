// ens_ffn.cu -- config 4 (S5'; reading A20 / A26): the ensemble layer's FFN branch, the MHA
// out-projection and the branch-sum LayerNorm in ONE kernel per 128-token tile:
//
//     acc = O Wo^T  +  sum_j ReLU(X W1_j^T + b1_j) W2_j^T          (j = 8 chunks of 128 hidden units)
//     Y   = LN_token(acc + (bo + b2) + S) * gamma + beta            (S = DCN branch, fp32; A26)
//
// Why: run as two GEMMs (FFN1 writing h, then [O | h] [Wo | W2]^T + LN) the FFN hidden h [B*64, 1024] bf16
// (1 GB at B = 8192) is written to and read back from HBM every layer.  Here each 128 x 128 chunk of h lives
// only in TMEM (fp32 accumulator, double-buffered) and shared memory (bf16, the A operand of the second MMA).
// The K order of acc is O (256) then h (1024) in 16-wide steps -- exactly the order of the [O | h] GEMM --
// and h is rounded to bf16 at the same point (A15), so the result is bit-identical to the two-GEMM path.
//
// Per CTA (persistent over token tiles), 10 warps:
//   warp 0      TMA producer: X tile (resident, 64 KB), O tile (64 KB, into the H region), and the weight ring
//               (3 x 32 KB): Wo k-blocks, then per chunk j the W1_j k-blocks and the W2_{j-1} k-blocks;
//   warp 1      TMEM allocator + MMA issuer: acc_out (TMEM cols 0-255) and acc_h[2] (256-383, 384-511);
//   warps 2-9   epilogue, 2 per TMEM lane quadrant: each h chunk -> +b1, ReLU, bf16 -> H[j % 2] (shared);
//               the 4 part-0 warps then run the LayerNorm epilogue (3 passes over TMEM) and TMA-store Y.
#include <cudaTypedefs.h>
#include <cuda_bf16.h>

#include "cvr_kernels.cuh"
#include "cvr_ptx.cuh"
#include "cvr_tile.cuh"

namespace cvr {
namespace {

using namespace tile;

constexpr int BM = 128, BK = 64, D = 256, F = 1024, HC = 128;  // model dims (A20), hidden chunk
constexpr int NCH = F / HC;                                       // 8 chunks
constexpr int SUB = BM * 64 * 2;                                  // 16 KB sub-tile (128 x 64 bf16)
constexpr int X_OFF = 0;                                          // X tile: 4 sub-tiles
constexpr int HB_OFF = 4 * SUB;                                   // O tile (4 subs) | H[2] (2 subs each) | Y staging
constexpr int RING_OFF = 8 * SUB;
constexpr int STAGE = 32 * 1024;
constexpr int STAGES = 3;
constexpr int BAR_OFF = RING_OFF + STAGES * STAGE;                // 224 KB
constexpr int SMEM = 1024 + BAR_OFF + 256;
constexpr int NT = 32 * 10;

__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) { ptx::mbar_wait(b, ph); }

__global__ void __launch_bounds__(NT, 1)
    ens_ffn_ln_kernel(const __grid_constant__ CUtensorMap tmX,    // x_l tokens [BT, 256], box {64, 128}
                      const __grid_constant__ CUtensorMap tmO,    // O = cat[:, :256] (ld D + F), box {64, 128}
                      const __grid_constant__ CUtensorMap tmW1,   // W1 [1024, 256], box {64, 128}
                      const __grid_constant__ CUtensorMap tmWc,   // [Wo | W2] [256, 1280], box {64, 256}
                      const __grid_constant__ CUtensorMap tmY,    // out tokens [BT, 256], box {64, 32}
                      const float* __restrict__ b1, const float* __restrict__ bcat, const float* __restrict__ S,
                      const float* __restrict__ gamma, const float* __restrict__ beta, int M) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + BAR_OFF);
  uint64_t* full = bars;                 // [3] ring
  uint64_t* empty = full + STAGES;       // [3]
  uint64_t* xfull = empty + STAGES;      // X tile landed
  uint64_t* xfree = xfull + 1;           // X no longer read (MMA commit)
  uint64_t* ofull = xfree + 1;           // O tile landed
  uint64_t* hbfree = ofull + 1;          // H region free for the next O (4 LN warps, after the Y store read)
  uint64_t* ofree = hbfree + 1;          // O consumed by the Wo MMAs: H may be written (MMA commit)
  uint64_t* hfull = ofree + 1;           // [2] acc_h ready (MMA commit)
  uint64_t* hempty = hfull + 2;          // [2] acc_h drained (8 warps)
  uint64_t* hready = hempty + 2;         // [2] H written (8 warps)
  uint64_t* hbuf_free = hready + 2;      // [2] H consumed by the W2 MMAs (MMA commit)
  uint64_t* outfull = hbuf_free + 2;     // acc_out complete (MMA commit)
  uint64_t* outempty = outfull + 1;      // acc_out drained (4 LN warps)
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(outempty + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_tiles = (M + BM - 1) / BM;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    ptx::mbar_init(xfull, 1);
    ptx::mbar_init(xfree, 1);
    ptx::mbar_init(ofull, 1);
    ptx::mbar_init(hbfree, 4);
    ptx::mbar_init(ofree, 1);
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&hfull[i], 1);
      ptx::mbar_init(&hempty[i], 8);
      ptx::mbar_init(&hready[i], 8);
      ptx::mbar_init(&hbuf_free[i], 1);
    }
    ptx::mbar_init(outfull, 1);
    ptx::mbar_init(outempty, 4);
    ptx::fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tmX);
    ptx::prefetch_tmap(&tmO);
    ptx::prefetch_tmap(&tmW1);
    ptx::prefetch_tmap(&tmWc);
    ptx::prefetch_tmap(&tmY);
  }
  if (warp == 1) ptx::tmem_alloc(tmem_holder, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  ptx::griddep_wait();
  ptx::griddep_launch();

  if (warp == 0) {
    if (lane == 0) {  // ================= TMA producer
      int g = 0;      // ring position
      auto ring = [&](const CUtensorMap* tm, int c0, int c1, uint32_t bytes) {
        const int s = g % STAGES;
        if (g >= STAGES) wait(&empty[s], ((g / STAGES) - 1) & 1);
        ptx::mbar_arrive_expect_tx(&full[s], bytes);
        ptx::tma_load_2d(smem + RING_OFF + s * STAGE, tm, &full[s], c0, c1);
        ++g;
      };
      int it = 0;
      for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++it) {
        const int m0 = tile * BM;
        if (it > 0) wait(xfree, (it - 1) & 1);
        ptx::mbar_arrive_expect_tx(xfull, 4 * SUB);
        for (int kb = 0; kb < 4; ++kb) ptx::tma_load_2d(smem + X_OFF + kb * SUB, &tmX, xfull, kb * BK, m0);
        if (it > 0) wait(hbfree, (it - 1) & 1);
        ptx::mbar_arrive_expect_tx(ofull, 4 * SUB);
        for (int kb = 0; kb < 4; ++kb) ptx::tma_load_2d(smem + HB_OFF + kb * SUB, &tmO, ofull, kb * BK, m0);
        for (int kb = 0; kb < 4; ++kb) ring(&tmWc, kb * BK, 0, 2 * SUB);             // Wo
        for (int j = 0; j <= NCH; ++j) {
          if (j < NCH)
            for (int kb = 0; kb < 4; ++kb) ring(&tmW1, kb * BK, j * HC, SUB);        // W1_j (128 rows)
          if (j > 0)
            for (int kb = 0; kb < 2; ++kb) ring(&tmWc, D + (j - 1) * HC + kb * BK, 0, 2 * SUB);  // W2_{j-1}
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ================= MMA issuer
      constexpr uint32_t id_out = ptx::idesc_bf16_f32(BM, D);
      constexpr uint32_t id_h = ptx::idesc_bf16_f32(BM, HC);
      const uint32_t acc_out = tmem, acc_h0 = tmem + 256;
      int g = 0, hc = 0, it = 0;
      auto stage = [&]() -> uint8_t* {
        const int s = g % STAGES;
        wait(&full[s], (g / STAGES) & 1);
        ptx::tc_fence_after();
        return smem + RING_OFF + s * STAGE;
      };
      auto release = [&]() { ptx::umma_commit(&empty[g % STAGES]); ++g; };
      for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++it) {
        wait(xfull, it & 1);
        wait(ofull, it & 1);
        if (it > 0) wait(outempty, (it - 1) & 1);
        ptx::tc_fence_after();
        for (int kb = 0; kb < 4; ++kb) {  // acc_out = O Wo^T
          const uint64_t bd = ptx::sdesc_kmajor_sw128(ptx::smem_u32(stage()));
          const uint64_t ad = ptx::sdesc_kmajor_sw128(ptx::smem_u32(smem + HB_OFF + kb * SUB));
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) ptx::umma_bf16_ss(acc_out, ad + 2 * k, bd + 2 * k, id_out, (kb | k) != 0);
          release();
        }
        ptx::umma_commit(ofree);
        for (int j = 0; j <= NCH; ++j) {
          if (j < NCH) {  // acc_h[b] = X W1_j^T
            const int u = hc + j, b = u & 1;
            if (u >= 2) wait(&hempty[b], ((u >> 1) - 1) & 1);
            ptx::tc_fence_after();
            for (int kb = 0; kb < 4; ++kb) {
              const uint64_t bd = ptx::sdesc_kmajor_sw128(ptx::smem_u32(stage()));
              const uint64_t ad = ptx::sdesc_kmajor_sw128(ptx::smem_u32(smem + X_OFF + kb * SUB));
#pragma unroll
              for (int k = 0; k < BK / 16; ++k)
                ptx::umma_bf16_ss(acc_h0 + b * HC, ad + 2 * k, bd + 2 * k, id_h, (kb | k) != 0);
              release();
            }
            ptx::umma_commit(&hfull[b]);
            if (j == NCH - 1) ptx::umma_commit(xfree);
          }
          if (j > 0) {  // acc_out += H_{j-1} W2_{j-1}^T
            const int u = hc + j - 1, b = u & 1;
            wait(&hready[b], (u >> 1) & 1);
            ptx::tc_fence_after();
            for (int kb = 0; kb < 2; ++kb) {
              const uint64_t bd = ptx::sdesc_kmajor_sw128(ptx::smem_u32(stage()));
              const uint64_t ad = ptx::sdesc_kmajor_sw128(ptx::smem_u32(smem + HB_OFF + (2 * b + kb) * SUB));
#pragma unroll
              for (int k = 0; k < BK / 16; ++k) ptx::umma_bf16_ss(acc_out, ad + 2 * k, bd + 2 * k, id_out, 1);
              release();
            }
            ptx::umma_commit(&hbuf_free[b]);
          }
        }
        ptx::umma_commit(outfull);
        hc += NCH;
      }
    }
  } else {  // ================= epilogue warps 2..9
    const int q = warp & 3, part = (warp - 2) >> 2, r = q * 32 + lane;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    int hc = 0, it = 0;
    for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++it) {
      const int m0 = tile * BM, m = m0 + r;
      const bool live = m < M;
      wait(ofree, it & 1);  // O consumed: the H buffers (over O) may be written
      for (int j = 0; j < NCH; ++j) {
        const int u = hc + j, b = u & 1;
        wait(&hfull[b], (u >> 1) & 1);
        ptx::tc_fence_after();
        if (u >= 2) wait(&hbuf_free[b], ((u >> 1) - 1) & 1);  // the W2 MMAs of chunk u-2 have read H[b]
        const uint32_t hsub = ptx::smem_u32(smem + HB_OFF + (2 * b + part) * SUB);
#pragma unroll
        for (int c = 0; c < 64; c += 32) {
          float v[32];
          ld32_tmem(tmem + 256 + b * HC + lane_off + part * 64 + c, v);
          const float4* b4 = reinterpret_cast<const float4*>(b1 + j * HC + part * 64 + c);
#pragma unroll
          for (int w = 0; w < 8; ++w) {
            const float4 bb = __ldg(b4 + w);
            v[4 * w] = fmaxf(v[4 * w] + bb.x, 0.f);
            v[4 * w + 1] = fmaxf(v[4 * w + 1] + bb.y, 0.f);
            v[4 * w + 2] = fmaxf(v[4 * w + 2] + bb.z, 0.f);
            v[4 * w + 3] = fmaxf(v[4 * w + 3] + bb.w, 0.f);
          }
          sts32_bf16(hsub, r, c >> 3, v);
        }
        ptx::tc_fence_before();
        ptx::fence_async_smem();  // generic-proxy H writes -> visible to the tensor core (async proxy)
        __syncwarp();
        if (lane == 0) {
          ptx::mbar_arrive(&hempty[b]);
          ptx::mbar_arrive(&hready[b]);
        }
      }
      hc += NCH;
      if (part == 0) {  // LayerNorm epilogue over acc_out (the 4 part-0 warps, one row per thread)
        wait(outfull, it & 1);
        ptx::tc_fence_after();
        const uint32_t trow = tmem + lane_off;
        float sum = 0.f;
#pragma unroll 1
        for (int c = 0; c < D; c += 32) {  // pass 1: y = acc + b + S, back into TMEM; row sum
          float v[32], x[32];
          ld32_tmem(trow + c, v);
          if (live) ld32_f32(S + (int64_t)m * D + c, x);
#pragma unroll
          for (int w = 0; w < 32; ++w) {
            v[w] = v[w] + __ldg(bcat + c + w) + (live ? x[w] : 0.f);
            sum += v[w];
          }
          st32_tmem(trow + c, v);
        }
        ptx::tmem_wait_st();
        const float mean = sum / (float)D;
        float var = 0.f;
#pragma unroll 1
        for (int c = 0; c < D; c += 32) {  // pass 2: centred second moment (biased variance, A20)
          float v[32];
          ld32_tmem(trow + c, v);
#pragma unroll
          for (int w = 0; w < 32; ++w) var = fmaf(v[w] - mean, v[w] - mean, var);
        }
        const float rstd = 1.f / sqrtf(var / (float)D + 1e-5f);
        // the Y staging reuses the H region: every W2 MMA of this tile has completed (outfull)
        const uint32_t ybase = ptx::smem_u32(smem + HB_OFF);
#pragma unroll 1
        for (int c = 0; c < D; c += 32) {  // pass 3: normalise, affine, bf16
          float v[32];
          ld32_tmem(trow + c, v);
#pragma unroll
          for (int w = 0; w < 32; ++w) v[w] = (v[w] - mean) * rstd * __ldg(gamma + c + w) + __ldg(beta + c + w);
          sts32_bf16(ybase + (c >> 6) * SUB, r, (c & 63) >> 3, v);
        }
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(outempty);
        ptx::fence_async_smem();
        __syncwarp();
        if (lane == 0) {
          for (int sb = 0; sb < 4; ++sb)
            ptx::tma_store_2d(&tmY, smem + HB_OFF + sb * SUB + q * 32 * 128, sb * 64, m0 + q * 32);
          ptx::bulk_commit();
          ptx::bulk_wait_read<0>();
          ptx::mbar_arrive(hbfree);  // the next tile's O may land in the H region
        }
      }
    }
    if (part == 0 && lane == 0) ptx::bulk_wait<0>();
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) ptx::tmem_dealloc(tmem, 512);
}

}  // namespace

cudaError_t launch_ens_ffn_ln(const EnsFfnArgs& a, cudaStream_t s) {
  if (a.M <= 0) return cudaSuccess;
  if (a.D != D || a.F != F) return cudaErrorInvalidValue;
  static bool attr_done = false;
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(ens_ffn_ln_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    if (e != cudaSuccess) return e;
    attr_done = true;
  }
  const int n_tiles = (a.M + BM - 1) / BM;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(n_tiles < a.num_sms ? n_tiles : a.num_sms);
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = SMEM;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = a.pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, ens_ffn_ln_kernel, *a.tmX, *a.tmO, *a.tmW1, *a.tmWc, *a.tmY, a.b1, a.bcat, a.S,
                            a.gamma, a.beta, a.M);
}

}  // namespace cvr
