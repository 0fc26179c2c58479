// cross_stack.cu -- the whole low-rank DCN-v2 cross stack (L layers = 2L GEMMs) in ONE persistent,
// dependency-driven tcgen05 kernel:
//
//     for l in 0..L-1:   t       = x_l V_l^T                      (GEMM 2l,   N = r)
//                        x_{l+1} = x0 * (t U_l^T + b_l) + x_l     (GEMM 2l+1, N = W)
//
// Why: at config 2's B = 4096 every GEMM is small (2-4 us); as separate launches each pays launch
// latency, TMEM/barrier setup, a pipeline fill and a drained tail.  Here all 2L GEMMs are one list of
// 128 x 64 tiles (GEMM-major, m-block-major inside a GEMM), dealt round-robin to one CTA per SM.  A tile of
// GEMM g for row block mb only needs the rows mb of GEMM g-1's output, so instead of a grid-wide barrier
// each (GEMM, row block) has a completion counter: the TMA producer spins (acquire) until the previous
// GEMM's counter for its row block is complete, so layer l+1 starts on early row blocks while layer l is
// still finishing late ones (wavefront), and weight tiles of the next GEMM stream in with no launch gap.
//
// Deadlock freedom: a CTA handles its tiles in global-list order and a tile depends only on tiles of the
// previous GEMM, which precede it in every CTA's list; all CTAs are resident (grid <= #SMs, 1 CTA/SM).
// Outputs are written with coalesced st.global from a swizzled smem staging tile, then __threadfence +
// a release atomic per warp; readers acquire, then fence.proxy.async before their TMA loads.
// Same MMAs, same K order and the same fp32 epilogue as the per-GEMM kernels: bit-identical results.
#include <cudaTypedefs.h>
#include <cuda_bf16.h>

#include "cvr_kernels.cuh"
#include "cvr_ptx.cuh"
#include "cvr_tile.cuh"

namespace cvr {
namespace {

using namespace tile;

constexpr int BM = 128, BK = 64, BN = 64;
constexpr int kThreads = 192;
constexpr int A_BYTES = BM * BK * 2;     // 16 KB
constexpr int B_BYTES = BN * BK * 2;     // 8 KB
constexpr int STAGE = A_BYTES + B_BYTES;
constexpr int SUB = BM * 64 * 2;         // 16 KB
constexpr int EIN_BYTES = 2 * SUB;       // x0 + x_l tiles per accumulator
constexpr int OUT_BYTES = SUB;           // staging per accumulator
constexpr int STAGES = 5;
constexpr int SMEM = 1024 + STAGES * STAGE + 2 * EIN_BYTES + 2 * OUT_BYTES + 256;
constexpr int TMEM_COLS = 2 * BN;

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_add(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Tile walk of one CTA: for every GEMM g in order, a contiguous, balanced chunk of g's tiles (m-major),
// so consecutive tiles of a CTA mostly share a row block and completion signals can be batched per
// (g, row block) run.
struct Walk {
  int g, j, j_end, nt, MB, n_gemm, cta, grid, ntv, ntu;
  __device__ __forceinline__ int tiles_of(int gg) const { return MB * ((gg & 1) ? ntu : ntv); }
  __device__ __forceinline__ void start(int gg) {
    g = gg;
    nt = (g & 1) ? ntu : ntv;
    const int T = tiles_of(g);
    j = (int)((int64_t)T * cta / grid);
    j_end = (int)((int64_t)T * (cta + 1) / grid);
  }
  __device__ __forceinline__ void init(int MB_, int L, int ntv_, int ntu_, int cta_, int grid_) {
    MB = MB_;
    n_gemm = 2 * L;
    ntv = ntv_;
    ntu = ntu_;
    cta = cta_;
    grid = grid_;
    start(0);
    settle();
  }
  __device__ __forceinline__ void settle() {  // skip empty chunks
    while (g < n_gemm && j >= j_end) {
      if (g + 1 >= n_gemm) {
        g = n_gemm;
        return;
      }
      start(g + 1);
    }
  }
  __device__ __forceinline__ bool valid() const { return g < n_gemm; }
  __device__ __forceinline__ int mb() const { return j / nt; }
  __device__ __forceinline__ int n() const { return j - (j / nt) * nt; }
  __device__ __forceinline__ void next() {
    ++j;
    settle();
  }
};

__global__ void __launch_bounds__(kThreads, 1)
    cross_stack_kernel(const __grid_constant__ CUtensorMap tmX0, const CrossStackTables* __restrict__ tbl,
                       const CrossStackArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = sA + STAGES * A_BYTES;
  uint8_t* sEin = sB + STAGES * B_BYTES;
  uint8_t* sOut = sEin + 2 * EIN_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sOut + 2 * OUT_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* efull = tempty + 2;
  uint64_t* eempty = efull + 2;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(eempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int M = a.M, W = a.W, R = a.R, L = a.L;
  const int MB = (M + BM - 1) / BM;
  const int ntv = R / BN, ntu = W / BN;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&tfull[b], 1);
      ptx::mbar_init(&tempty[b], 4);
      ptx::mbar_init(&efull[b], 1);
      ptx::mbar_init(&eempty[b], 4);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tmX0);
    ptx::prefetch_tmap(&tbl->xa);
    ptx::prefetch_tmap(&tbl->xb);
    ptx::prefetch_tmap(&tbl->t);
  }
  if (warp == 1) ptx::tmem_alloc(tmem_holder, TMEM_COLS);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  ptx::griddep_wait();
  if (a.dbg && threadIdx.x == 0) a.dbg[blockIdx.x * 32 + 31] = gtimer();

  // x_l map for layer l (l = 0: x0; the outputs alternate x_a, x_b)
  auto xl_map = [&](int l) -> const CUtensorMap* { return l == 0 ? &tmX0 : ((l - 1) % 2 == 0 ? &tbl->xa : &tbl->xb); };

  if (warp == 0) {
    if (lane == 0) {  // ================= producer: dependencies + TMA
      int gk = 0, ue = 0;  // ue: U tiles so far (the x0 / x_l epilogue buffers cycle over U tiles only)
      Walk w;
      w.init(MB, L, ntv, ntu, blockIdx.x, gridDim.x);
      int ready_g = -1, ready_mb = -1;
      for (; w.valid(); w.next()) {
        const int g = w.g, l = g >> 1, kind = g & 1, mb = w.mb();
        const int m0 = mb * BM, n0 = w.n() * BN;
        if (g > 0 && (g != ready_g || mb != ready_mb)) {  // rows mb of GEMM g-1 must be complete
          const int need = 4 * (kind == 0 ? ntu : ntv);
          const int* cnt = a.done + (g - 1) * MB + mb;
          while (ld_acquire(cnt) < need) __nanosleep(32);
          ptx::fence_async_global();
          if (a.dbg && g != ready_g) a.dbg[blockIdx.x * 32 + 16 + g] = gtimer();
          ready_g = g;
          ready_mb = mb;
        }
        const CUtensorMap* A = kind == 0 ? xl_map(l) : &tbl->t;
        const CUtensorMap* Bm = kind == 0 ? &tbl->V[l] : &tbl->U[l];
        if (kind == 1) {
          const int b = ue & 1;
          if (ue >= 2) ptx::mbar_wait(&eempty[b], ((ue >> 1) - 1) & 1);
          ptx::mbar_arrive_expect_tx(&efull[b], EIN_BYTES);
          ptx::tma_load_2d(sEin + b * EIN_BYTES, &tmX0, &efull[b], n0, m0);
          ptx::tma_load_2d(sEin + b * EIN_BYTES + SUB, xl_map(l), &efull[b], n0, m0);
          ++ue;
        }
        const int nk = (kind == 0 ? W : R) / BK;
        for (int kb = 0; kb < nk; ++kb, ++gk) {
          const int s = gk % STAGES;
          if (gk >= STAGES) ptx::mbar_wait(&empty[s], ((gk / STAGES) - 1) & 1);
          ptx::mbar_arrive_expect_tx(&full[s], STAGE);
          ptx::tma_load_2d(sA + s * A_BYTES, A, &full[s], kb * BK, m0);
          ptx::tma_load_2d(sB + s * B_BYTES, Bm, &full[s], kb * BK, n0);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ================= MMA issuer
      constexpr uint32_t idesc = ptx::idesc_bf16_f32(BM, BN);
      int gk = 0, it = 0;
      Walk w;
      w.init(MB, L, ntv, ntu, blockIdx.x, gridDim.x);
      for (; w.valid(); w.next(), ++it) {
        const int kind = w.g & 1;
        const int b = it & 1;
        if (it >= 2) ptx::mbar_wait(&tempty[b], ((it >> 1) - 1) & 1);
        ptx::tc_fence_after();
        const uint32_t acc = tmem + b * BN;
        const int nk = (kind == 0 ? W : R) / BK;
        for (int kb = 0; kb < nk; ++kb, ++gk) {
          const int s = gk % STAGES;
          ptx::mbar_wait(&full[s], (gk / STAGES) & 1);
          ptx::tc_fence_after();
          const uint64_t ad = ptx::sdesc_kmajor_sw128(ptx::smem_u32(sA + s * A_BYTES));
          const uint64_t bd = ptx::sdesc_kmajor_sw128(ptx::smem_u32(sB + s * B_BYTES));
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) ptx::umma_bf16_ss(acc, ad + 2 * k, bd + 2 * k, idesc, (kb | k) != 0);
          ptx::umma_commit(&empty[s]);
        }
        ptx::umma_commit(&tfull[b]);
      }
    }
  } else {  // ================= epilogue warps 2..5 (TMEM quadrant q = rows 32q .. 32q+31)
    const int q = warp & 3, r = q * 32 + lane;
    int it = 0, ue = 0;
    Walk w;
    w.init(MB, L, ntv, ntu, blockIdx.x, gridDim.x);
    int pend = 0;  // tiles of the current (g, mb) run whose signal is not yet published
    for (; w.valid(); ++it) {
      struct {
        int g, l, kind, mb;
      } t = {w.g, w.g >> 1, w.g & 1, w.mb()};
      const int m0 = t.mb * BM, n0 = w.n() * BN;
      const int b = it & 1, be = ue & 1;
      ptx::mbar_wait(&tfull[b], (it >> 1) & 1);
      ptx::tc_fence_after();
      const uint32_t trow = tmem + b * BN + ((uint32_t)(q * 32) << 16);
      const uint32_t ob = ptx::smem_u32(sOut + b * OUT_BYTES);
      const uint32_t eb = ptx::smem_u32(sEin + be * EIN_BYTES);
      if (t.kind == 1) ptx::mbar_wait(&efull[be], (ue >> 1) & 1);
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        float v[32];
        ld32_tmem(trow + c, v);
        if (t.kind == 1) {
          const float* bias = a.bias[t.l] + n0 + c;
          float x0v[32], xlv[32];
          lds32_bf16(eb, r, c >> 3, x0v);
          lds32_bf16(eb + SUB, r, c >> 3, xlv);
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = x0v[j] * (v[j] + __ldg(bias + j)) + xlv[j];
        }
        sts32_bf16(ob, r, c >> 3, v);
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        ptx::mbar_arrive(&tempty[b]);
        if (t.kind == 1) ptx::mbar_arrive(&eempty[be]);
      }
      if (t.kind == 1) ++ue;
      // coalesced copy-out of this warp's 32 rows: 8 lanes per 128-byte row, 4 rows per instruction
      __nv_bfloat16* dst;
      int64_t ld;
      if (t.kind == 0) {
        dst = a.t;
        ld = R;
      } else {
        dst = (t.l % 2 == 0) ? a.xa : a.xb;
        ld = W;
      }
#pragma unroll
      for (int p = 0; p < 8; ++p) {
        const int rr = q * 32 + p * 4 + (lane >> 3), ch = lane & 7;
        const uint4 v = lds128(swz(ob, rr, ch));
        if (m0 + rr < M) *reinterpret_cast<uint4*>(dst + (int64_t)(m0 + rr) * ld + n0 + ch * 8) = v;
      }
      // publish the (g, mb) run when it ends: one fence per run instead of one per tile.  A run never
      // outlives its GEMM chunk, so the CTA's own later tiles (which may depend on it) cannot deadlock.
      ++pend;
      w.next();
      if (!w.valid() || w.g != t.g || w.mb() != t.mb) {
        __syncwarp();
        __threadfence();
        if (lane == 0) red_release_add(a.done + t.g * MB + t.mb, pend);
        pend = 0;
        if (a.dbg && lane == 0 && q == 0) a.dbg[blockIdx.x * 32 + t.g] = gtimer();
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::griddep_launch();
  if (warp == 1) ptx::tmem_dealloc(tmem, TMEM_COLS);
}

}  // namespace

cudaError_t launch_cross_stack(const CUtensorMap* tmX0, const CrossStackTables* d_tables, const CrossStackArgs& a,
                               cudaStream_t s) {
  if (a.M <= 0) return cudaSuccess;
  if (a.R % BN || a.W % BN || a.L < 1 || a.L > kMaxLayers) return cudaErrorInvalidValue;
  static bool attr_done = false;
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(cross_stack_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    if (e != cudaSuccess) return e;
    attr_done = true;
  }
  const int MB = (a.M + BM - 1) / BM;
  cudaError_t e = cudaMemsetAsync(a.done, 0, sizeof(int) * 2 * a.L * MB, s);
  if (e != cudaSuccess) return e;
  const int n_tiles = a.L * MB * (a.R / BN + a.W / BN);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(n_tiles < a.num_sms ? n_tiles : a.num_sms);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = SMEM;
  cfg.stream = s;
  cfg.numAttrs = 0;
  return cudaLaunchKernelEx(&cfg, cross_stack_kernel, *tmX0, d_tables, a);
}

}  // namespace cvr
