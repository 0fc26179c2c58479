// ffn_fused.cu -- config 4's token-wise FFN, attention out-projection and branch-sum LayerNorm as ONE tcgen05
// kernel (SURVEY.md §8(a) S5', reading A20):
//
//   h   = ReLU(X W1^T + b1)                                     [128 tokens x F] per tile, never stored
//   y   = [O | h] [Wo | W2]^T + (bo + b2) + S                   S = the layer's DCN branch (fp32)
//   X'  = LN_row(y) * gamma + beta                              bf16
//
// The unfused path runs FFN1 (writes h, 1 GB per layer at B = 8192) and one [O | h] GEMM with the LN epilogue
// (reads it back): both HBM-bound.  Here each CTA owns 128 tokens at a time and walks the hidden dimension in
// chunks of FH = 128: FFN1 of chunk c lands in one of two TMEM accumulators, the epilogue warps turn it into the
// bf16 A operand of chunk c's FFN2 in shared memory, and FFN2 accumulates into the output accumulator -- h only
// ever lives in TMEM and shared memory.  The output accumulator sees the same K order as the unfused GEMM (O's 256
// columns, then h in chunk order), every rounding point is the same (h + b1 -> ReLU -> bf16; (acc + b) + S; LN in
// fp32), so the scores are bit-identical to the unfused path.
//
// Roles (224 threads): warp 0 streams the weight / O ring (TMA), warp 1 allocates TMEM and issues the MMAs, warps
// 2-5 are the epilogue (TMEM lane quadrant warp % 4: 32 tokens each), warp 6 loads the resident X tile.
// Shared memory: X [4 k-blocks of 128 x 64] 64 KB | h chunk [2 k-blocks] 32 KB | ring 3 x 32 KB (W1 chunk k-block
// 16 KB, W2 k-block 256 x 64 = 32 KB, out-projection [O k-block | Wo half k-block]) | per-warp S input ring / output
// staging 4 x 2 x 4 KB.  TMEM: output accumulator [0, 256), FFN1 accumulators [256, 384) and [384, 512).
#include "cvr_kernels.cuh"
#include "cvr_ptx.cuh"
#include "cvr_tile.cuh"

namespace cvr {
namespace {

using namespace tile;

constexpr int FM = 128;                 // tokens per tile
constexpr int FD = 256;                 // model width D (output columns)
constexpr int FH = 128;                 // hidden chunk
constexpr int SUBT = FM * 64 * 2;       // one [128 x 64] bf16 k-block (16 KB)
constexpr int RING = 3;
constexpr int SLOT = 32768;
constexpr int OFF_X = 0;
constexpr int OFF_H = OFF_X + 4 * SUBT;
constexpr int OFF_R = OFF_H + 2 * SUBT;
constexpr int OFF_S = OFF_R + RING * SLOT;
constexpr int OFF_BAR = OFF_S + 4 * 2 * 4096;
constexpr int FFN_SMEM = 1024 + OFF_BAR + 256;
constexpr int FFN_THREADS = 7 * 32;

__global__ void __launch_bounds__(FFN_THREADS, 1)
    ffn_fused_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmO,
                     const __grid_constant__ CUtensorMap tmW1, const __grid_constant__ CUtensorMap tmW2,
                     const __grid_constant__ CUtensorMap tmWo, const __grid_constant__ CUtensorMap tmS,
                     const __grid_constant__ CUtensorMap tmOut, const FfnArgs g) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sX = smem + OFF_X;
  uint8_t* sH = smem + OFF_H;
  uint8_t* sR = smem + OFF_R;
  uint8_t* sS = smem + OFF_S;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
  uint64_t* rfull = bars;            // [RING]
  uint64_t* rempty = rfull + RING;   // [RING]
  uint64_t* xfull = rempty + RING;
  uint64_t* xempty = xfull + 1;
  uint64_t* afull = xempty + 1;      // [2] FFN1 accumulator ready
  uint64_t* aempty = afull + 2;      // [2] FFN1 accumulator drained (4 warps)
  uint64_t* hfull = aempty + 2;      // h chunk staged (4 warps)
  uint64_t* hempty = hfull + 1;      // [2] h k-block kb read by FFN2 (the epilogue refills k-block 0 while FFN2
                                     // still reads k-block 1)
  uint64_t* ofull = hempty + 2;      // output accumulator complete
  uint64_t* oempty = ofull + 1;      // output accumulator drained (4 warps)
  uint64_t* sfull = oempty + 1;      // [4 warps][2] S chunk landed
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(sfull + 8);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int M = g.call ? g.call->B * g.m_mult : g.M;  // tokens
  const int F = g.F, nch = F / FH;
  const int n_tiles = (M + FM - 1) / FM;

  if (threadIdx.x == 0) {
    for (int s = 0; s < RING; ++s) {
      ptx::mbar_init(&rfull[s], 1);
      ptx::mbar_init(&rempty[s], 1);
    }
    ptx::mbar_init(xfull, 1);
    ptx::mbar_init(xempty, 1);
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&afull[b], 1);
      ptx::mbar_init(&aempty[b], 4);
    }
    ptx::mbar_init(hfull, 4);
    ptx::mbar_init(&hempty[0], 1);
    ptx::mbar_init(&hempty[1], 1);
    ptx::mbar_init(ofull, 1);
    ptx::mbar_init(oempty, 4);
    for (int i = 0; i < 8; ++i) ptx::mbar_init(&sfull[i], 1);
    ptx::fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tmW1);
    ptx::prefetch_tmap(&tmW2);
    ptx::prefetch_tmap(&tmWo);
    ptx::prefetch_tmap(&tmO);
  }
  if (warp == 1) ptx::tmem_alloc(tmem_holder, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  ptx::griddep_wait();  // X, O and S were written by the previous kernels
  ptx::griddep_launch();

  if (warp == 0) {
    // ================= ring producer: per tile, in the MMA warp's order: W1(0), W1(1), out-projection, W2(0), then
    // W1(c), W2(c-1) for c = 2 .. nch-1, and W2(nch-1)
    if (lane == 0) {
      int gk = 0;
      auto slot = [&]() -> uint8_t* {
        const int s = gk % RING;
        if (gk >= RING) ptx::mbar_wait(&rempty[s], ((gk / RING) - 1) & 1);
        return sR + s * SLOT;
      };
      auto w1 = [&](int c) {
        for (int kb = 0; kb < FD / 64; ++kb) {
          uint8_t* d = slot();
          const int s = gk % RING;
          ptx::mbar_arrive_expect_tx(&rfull[s], SUBT);
          ptx::tma_load_2d(d, &tmW1, &rfull[s], kb * 64, c * FH);
          ++gk;
        }
      };
      auto w2 = [&](int c) {
        for (int kb = 0; kb < FH / 64; ++kb) {
          uint8_t* d = slot();
          const int s = gk % RING;
          ptx::mbar_arrive_expect_tx(&rfull[s], 2 * SUBT);
          ptx::tma_load_2d(d, &tmW2, &rfull[s], FD + c * FH + kb * 64, 0);
          ++gk;
        }
      };
      for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        const int m0 = tile * FM;
        w1(0);
        if (nch > 1) w1(1);
        for (int h = 0; h < 2; ++h)  // out-projection: [O k-block | Wo rows 128 h .. +128 k-block]
          for (int kb = 0; kb < FD / 64; ++kb) {
            uint8_t* d = slot();
            const int s = gk % RING;
            ptx::mbar_arrive_expect_tx(&rfull[s], 2 * SUBT);
            ptx::tma_load_2d(d, &tmO, &rfull[s], kb * 64, m0);
            ptx::tma_load_2d(d + SUBT, &tmWo, &rfull[s], kb * 64, h * 128);
            ++gk;
          }
        w2(0);
        for (int c = 2; c < nch; ++c) {
          w1(c);
          w2(c - 1);
        }
        if (nch > 1) w2(nch - 1);
      }
    }
  } else if (warp == 6) {
    // ================= X producer: the tile's 128 tokens x 256, resident while its FFN1 chunks run
    if (lane == 0) {
      int it = 0;
      for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++it) {
        if (it >= 1) ptx::mbar_wait(xempty, (it - 1) & 1);
        ptx::mbar_arrive_expect_tx(xfull, 4 * SUBT);
        for (int kb = 0; kb < 4; ++kb) ptx::tma_load_2d(sX + kb * SUBT, &tmX, xfull, kb * 64, tile * FM);
      }
    }
  } else if (warp == 1) {
    // ================= MMA issuer
    if (lane == 0) {
      constexpr uint32_t id128 = ptx::idesc_bf16_f32(128, 128), id256 = ptx::idesc_bf16_f32(128, 256);
      int gk = 0, ca = 0, hc = 0, it = 0;
      auto full_slot = [&]() -> uint32_t {
        const int s = gk % RING;
        ptx::mbar_wait(&rfull[s], (gk / RING) & 1);
        ptx::tc_fence_after();
        return ptx::smem_u32(sR + s * SLOT);
      };
      auto release = [&]() {
        ptx::umma_commit(&rempty[gk % RING]);
        ++gk;
      };
      auto ffn1 = [&](int c) {  // acc1[b] = X W1_c^T
        const int b = ca & 1;
        if (ca >= 2) ptx::mbar_wait(&aempty[b], ((ca >> 1) - 1) & 1);
        ptx::tc_fence_after();
        const uint32_t d = tmem + 256 + 128 * b;
        for (int kb = 0; kb < FD / 64; ++kb) {
          const uint32_t sb = full_slot();
          const uint64_t ad = ptx::sdesc_kmajor_sw128(ptx::smem_u32(sX + kb * SUBT));
          const uint64_t bd = ptx::sdesc_kmajor_sw128(sb);
#pragma unroll
          for (int k = 0; k < 4; ++k) ptx::umma_bf16_ss(d, ad + 2 * k, bd + 2 * k, id128, (kb | k) != 0);
          release();
        }
        ptx::umma_commit(&afull[b]);
        ++ca;
        if (c == nch - 1) ptx::umma_commit(xempty);  // the tile's last read of X
      };
      auto ffn2 = [&](int c) {  // out += h_c W2_c^T
        ptx::mbar_wait(hfull, hc & 1);
        ptx::tc_fence_after();
        for (int kb = 0; kb < FH / 64; ++kb) {
          const uint32_t sb = full_slot();
          const uint64_t ad = ptx::sdesc_kmajor_sw128(ptx::smem_u32(sH + kb * SUBT));
          const uint64_t bd = ptx::sdesc_kmajor_sw128(sb);
#pragma unroll
          for (int k = 0; k < 4; ++k) ptx::umma_bf16_ss(tmem, ad + 2 * k, bd + 2 * k, id256, 1);
          release();
          ptx::umma_commit(&hempty[kb]);
        }
        ++hc;
        (void)c;
      };
      for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++it) {
        ptx::mbar_wait(xfull, it & 1);
        ptx::tc_fence_after();
        ffn1(0);
        if (nch > 1) ffn1(1);
        // out-projection first (the unfused GEMM's K order: O's columns, then h): the output accumulator must have
        // been drained by the previous tile's LN epilogue
        if (it >= 1) ptx::mbar_wait(oempty, (it - 1) & 1);
        ptx::tc_fence_after();
        for (int h = 0; h < 2; ++h)
          for (int kb = 0; kb < FD / 64; ++kb) {
            const uint32_t sb = full_slot();
            const uint64_t ad = ptx::sdesc_kmajor_sw128(sb);
            const uint64_t bd = ptx::sdesc_kmajor_sw128(sb + SUBT);
#pragma unroll
            for (int k = 0; k < 4; ++k) ptx::umma_bf16_ss(tmem + 128 * h, ad + 2 * k, bd + 2 * k, id128, (kb | k) != 0);
            release();
          }
        ffn2(0);
        for (int c = 2; c < nch; ++c) {
          ffn1(c);
          ffn2(c - 1);
        }
        if (nch > 1) ffn2(nch - 1);
        ptx::umma_commit(ofull);
      }
    }
  } else {
    // ================= epilogue warps 2-5: TMEM lane quadrant q -> tokens 32 q .. 32 q + 31 of the tile
    const int q = warp & 3, wq = warp - 2;
    const int r = q * 32 + lane;
    const uint32_t lanebase = (uint32_t)(q * 32) << 16;
    uint8_t* myS = sS + wq * 2 * 4096;
    int ca = 0, hc = 0, it = 0, sk = 0;
    for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++it) {
      const int m0 = tile * FM;
      if (lane == 0) {  // the tile's first two S chunks (32 tokens x 32 columns fp32 each)
        ptx::fence_async_smem();
        for (int i = 0; i < 2; ++i) {
          const int b = (sk + i) & 1;
          ptx::mbar_arrive_expect_tx(&sfull[wq * 2 + b], 4096);
          ptx::tma_load_2d(myS + b * 4096, &tmS, &sfull[wq * 2 + b], 32 * i, m0 + q * 32);
        }
      }
      // ---- hidden chunks: h = ReLU(acc1 + b1) -> bf16 A operand of FFN2 (same rounding as EPI_BIAS_RELU)
      for (int c = 0; c < nch; ++c) {
        const int b = ca & 1;
        ptx::mbar_wait(&afull[b], (ca >> 1) & 1);
        ptx::tc_fence_after();
        const uint32_t trow = tmem + 256 + 128 * b + lanebase;
        const uint32_t hbase = ptx::smem_u32(sH);
#pragma unroll 1
        for (int cc = 0; cc < FH; cc += 32) {
          float v[32];
          ld32_tmem(trow + cc, v);
          const float4* b4 = reinterpret_cast<const float4*>(g.b1 + c * FH + cc);
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const float4 bb = __ldg(b4 + u);
            v[4 * u] = fmaxf(v[4 * u] + bb.x, 0.f);
            v[4 * u + 1] = fmaxf(v[4 * u + 1] + bb.y, 0.f);
            v[4 * u + 2] = fmaxf(v[4 * u + 2] + bb.z, 0.f);
            v[4 * u + 3] = fmaxf(v[4 * u + 3] + bb.w, 0.f);
          }
          // FFN2 of the previous chunk has read this h k-block (the first wait per k-block; the accumulator read and
          // the bias work above already overlap it)
          if ((cc & 63) == 0 && hc >= 1) ptx::mbar_wait(&hempty[cc >> 6], (hc - 1) & 1);
          sts32_bf16(hbase + (cc >> 6) * SUBT, r, (cc & 63) >> 3, v);
        }
        ptx::tc_fence_before();
        ptx::fence_async_smem();  // the generic-proxy h stores -> visible to the tensor core
        __syncwarp();
        if (lane == 0) {
          ptx::mbar_arrive(&aempty[b]);
          ptx::mbar_arrive(hfull);
        }
        ++ca;
        ++hc;
      }
      // ---- LN epilogue (EPI_SUM_LN's arithmetic): y = (acc + b) + S, mean, centred variance, affine, bf16
      ptx::mbar_wait(ofull, it & 1);
      ptx::tc_fence_after();
      const uint32_t orow = tmem + lanebase;
      float sum = 0.f;
#pragma unroll 1
      for (int i = 0; i < FD / 32; ++i) {
        const int c = 32 * i, k = sk + i, b = k & 1;
        float v[32], x[32];
        ld32_tmem(orow + c, v);
        ptx::mbar_wait(&sfull[wq * 2 + b], (k >> 1) & 1);
        const uint32_t xt = ptx::smem_u32(myS + b * 4096);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const uint4 w4 = lds128(xt + lane * 128 + ((u ^ (lane & 7)) << 4));
          x[4 * u] = __uint_as_float(w4.x);
          x[4 * u + 1] = __uint_as_float(w4.y);
          x[4 * u + 2] = __uint_as_float(w4.z);
          x[4 * u + 3] = __uint_as_float(w4.w);
        }
        __syncwarp();
        if (lane == 0 && i + 2 < FD / 32) {  // refill this buffer with chunk i + 2
          ptx::fence_async_smem();
          ptx::mbar_arrive_expect_tx(&sfull[wq * 2 + b], 4096);
          ptx::tma_load_2d(myS + b * 4096, &tmS, &sfull[wq * 2 + b], c + 64, m0 + q * 32);
        }
        const float4* bc4 = reinterpret_cast<const float4*>(g.bcat + c);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const float4 bb = __ldg(bc4 + u);
          v[4 * u] = v[4 * u] + bb.x + x[4 * u];
          v[4 * u + 1] = v[4 * u + 1] + bb.y + x[4 * u + 1];
          v[4 * u + 2] = v[4 * u + 2] + bb.z + x[4 * u + 2];
          v[4 * u + 3] = v[4 * u + 3] + bb.w + x[4 * u + 3];
        }
#pragma unroll
        for (int j = 0; j < 32; ++j) sum += v[j];
        st32_tmem(orow + c, v);
      }
      sk += FD / 32;
      ptx::tmem_wait_st();
      const float mean = sum / (float)FD;
      float var = 0.f;
#pragma unroll 1
      for (int c = 0; c < FD; c += 32) {
        float v[32];
        ld32_tmem(orow + c, v);
#pragma unroll
        for (int j = 0; j < 32; ++j) var = fmaf(v[j] - mean, v[j] - mean, var);
      }
      const float rstd = 1.f / sqrtf(var / (float)FD + 1e-5f);
      // normalise -> bf16 -> this warp's staging (its two S buffers, free now) -> TMA store of 32 tokens x 64
#pragma unroll 1
      for (int blk = 0; blk < FD / 64; ++blk) {
        uint8_t* st = myS + (blk & 1) * 4096;
        if (blk >= 2) {
          if (lane == 0) ptx::bulk_wait_read<1>();  // the store from this buffer two blocks ago has read it
          __syncwarp();
        }
        const uint32_t sb = ptx::smem_u32(st);
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          const int c = 64 * blk + 32 * half;
          float v[32];
          ld32_tmem(orow + c, v);
          const float4* ga4 = reinterpret_cast<const float4*>(g.gamma + c);
          const float4* be4 = reinterpret_cast<const float4*>(g.beta + c);
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const float4 ga = __ldg(ga4 + u), be = __ldg(be4 + u);
            v[4 * u] = (v[4 * u] - mean) * rstd * ga.x + be.x;
            v[4 * u + 1] = (v[4 * u + 1] - mean) * rstd * ga.y + be.y;
            v[4 * u + 2] = (v[4 * u + 2] - mean) * rstd * ga.z + be.z;
            v[4 * u + 3] = (v[4 * u + 3] - mean) * rstd * ga.w + be.w;
          }
          sts32_bf16(sb, lane, half * 4, v);
        }
        ptx::fence_async_smem();
        __syncwarp();
        if (lane == 0) {
          ptx::tma_store_2d(&tmOut, st, 64 * blk, m0 + q * 32);
          ptx::bulk_commit();
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        ptx::mbar_arrive(oempty);      // the output accumulator is free for the next tile's out-projection
        ptx::bulk_wait_read<0>();      // the staging (= next tile's S buffers) has been read by the stores
      }
      __syncwarp();
    }
    if (lane == 0) ptx::bulk_wait<0>();  // this warp's output stores complete before the CTA exits
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) ptx::tmem_dealloc(tmem, 512);
}

}  // namespace

cudaError_t launch_ffn_fused(const FfnArgs& g, cudaStream_t s) {
  if (g.F % FH || g.F / FH < 2 || g.D != FD) return cudaErrorInvalidValue;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(ffn_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, FFN_SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int tiles = (g.M + FM - 1) / FM;  // (executor graphs: g.M = max rows; the kernel reads the batch's rows)
  const int grid = tiles < g.num_sms ? tiles : g.num_sms;
  if (grid <= 0) return cudaSuccess;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(FFN_THREADS);
  cfg.dynamicSmemBytes = FFN_SMEM;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = g.pdl ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, ffn_fused_kernel, *g.tmX, *g.tmO, *g.tmW1, *g.tmW2, *g.tmWo, *g.tmS, *g.tmOut, g);
}

}  // namespace cvr
