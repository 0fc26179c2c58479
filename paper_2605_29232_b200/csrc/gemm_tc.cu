// gemm_tc.cu -- K4: bf16 GEMM on the 5th-generation tensor cores (tcgen05 + TMEM + TMA) with the
// dense stage's elementwise work fused into the epilogue:
//
//   EPI_STORE      C = A B^T                         t = x_l V_l^T
//   EPI_CROSS      C = x0 * (A B^T + b) + x_l        x_{l+1} = x0 * (U_l t + b_l) + x_l
//                                                    (PAPER.md:225 low-rank DCNv2; A9 bias)
//   EPI_BIAS_RELU  C = ReLU(A B^T + b)               MLP tower
//   EPI_HEAD       s = sigmoid(ReLU(A B^T + b) . m + c)   last MLP layer + head, h never stored
//                                                    (BASELINE.json north star)
//   EPI_MASK       C = (A B^T + b) * x_l             MaskNet block x_{l+1} = (U_l h + b_l) * x_l with
//                                                    h = ReLU(V_l x0' + c_l) (A27)
//
// Design (persistent, warp-specialised, one CTA per SM):
//   * A [M, K] and B [N, K] bf16, K-major, moved by TMA into 128-byte-swizzled shared memory
//     (BK = 64 elements = one swizzle atom) through a STAGES-deep full/empty mbarrier ring.
//   * warp 0 = TMA producer (also loads the x0 / x_l epilogue tiles of EPI_CROSS by TMA);
//     warp 1 = TMEM allocator + single-thread tcgen05.mma issuer (M=128, N=BN, K=16);
//     warps 2-5 = epilogue, each owning a 32-lane TMEM quadrant (= 32 rows of the tile).
//   * Two TMEM accumulators (2 x BN columns): the epilogue of tile i overlaps the MMAs of
//     tile i+1.  Output tiles are staged in swizzled shared memory and written by TMA stores.
//   * Tiles are visited n-fastest so CTAs working at the same time share the A row block in L2.
//   * Programmatic dependent launch: the prologue (barrier init, TMEM alloc, descriptor
//     prefetch) runs before griddepcontrol.wait, overlapping the previous kernel's tail; the
//     dependent launch is triggered right after the wait.
//   * No split-K: every row's result depends only on that row, in a fixed K order, so scores are
//     batch-invariant.
#include <cudaTypedefs.h>
#include <cuda_bf16.h>

#include "cvr_attn.cuh"
#include "cvr_kernels.cuh"
#include "cvr_ptx.cuh"
#include "cvr_tile.cuh"

namespace cvr {
namespace {

constexpr int BM = 128;
constexpr int BK = 64;

constexpr int kSmemBudget = 225 * 1024;

template <int EPI>
struct EpiTraits {
  static constexpr bool kSmemOut = EPI == EPI_STORE || EPI == EPI_BIAS_RELU || EPI == EPI_CROSS || EPI == EPI_BIAS ||
                                   EPI == EPI_SUM_LN || EPI == EPI_MASK;
  static constexpr bool kEin = EPI == EPI_CROSS || EPI == EPI_CROSS_F32 || EPI == EPI_MASK;  // x0 / x_l tiles (TMA)
  static constexpr int kEinTensors = EPI == EPI_MASK ? 1 : 2;                                  // MASK: x_l only
  static constexpr bool kBias = EPI != EPI_STORE;
};

// EIN slots (EPI_CROSS at BN = 192): x0 / x_l come as 64-column sub-tile pairs, one slot per sub-tile
// position j, fed by a dedicated producer warp; 3 epilogue warps per TMEM lane quadrant, warp part j owning
// sub-tile j, write x_{l+1} in place over x_l and TMA-store it from there (no separate output staging):
// 96 KB of epilogue buffers instead of 2 x 96 + 48, and the three sub-tiles are finished in parallel.
template <int BN, int EPI, int CG>
constexpr bool ein_ring() { return EPI == EPI_CROSS && BN == 192; }

template <int BN, int EPI, int CG = 1, int EW = 4>
struct Cfg {
  static constexpr int A_BYTES = BM * BK * 2;       // 16 KB
  static constexpr int B_BYTES = (BN / CG) * BK * 2;  // CG = 2: each CTA of the pair holds half of B
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int SUB = BM * 64 * 2;           // one 128 x 64 bf16 sub-tile (16 KB)
  static constexpr int NSUB = BN / 64;
  static constexpr int OUT_BUFS = BN >= 192 ? 1 : 2;
  static constexpr bool RING = ein_ring<BN, EPI, CG>();
  static constexpr int RING_SLOTS = 3;

  // epilogue warps per TMEM lane quadrant: the epilogue of a CTA's last tile is exposed (one tile per CTA at
  // B = 4096), so plain stores split the tile's 64-column sub-tiles over up to 4 warps per quadrant
  // (EPI_HEAD too: each warp's partial dot product over its 64-column sub-tiles, summed in column order)
  static constexpr bool SPLIT = EPI == EPI_STORE || EPI == EPI_BIAS_RELU || EPI == EPI_BIAS || EPI == EPI_HEAD ||
                                EPI == EPI_CROSS_F32;
  // EW caps the split: EW = 1 when each CTA runs several tiles (the epilogue then overlaps the next tile's
  // mainloop anyway) keeps the CTA at 7 warps, leaving registers for co-resident embedding CTAs
  // EPI_ATTN: 8 epilogue warps = 2 examples x 4 groups of 16 query rows (one attention warp each)
  static constexpr bool ATTN = EPI == EPI_ATTN;
  // EPI_ATTN_TC: two groups of 4 epilogue warps (one per TMEM lane quadrant) take alternate tiles (group = the
  // tile's accumulator), each with its own attention-MMA warp and its own Q | K | V staging [3][128 x 64] bf16 in the
  // 128-byte-swizzled UMMA layout (Q doubles as the O staging of the TMA store); P never touches shared memory:
  // the softmax writes it back into TMEM as the A operand of O = P V
  static constexpr bool ATTN_TC = EPI == EPI_ATTN_TC;
  // ATTN: two groups of 8 epilogue warps take alternate tiles (accumulator a = group), each with its own staging,
  // so one tile's attention overlaps the next one's
  static constexpr int ATT_GROUPS = 2;
  // (EPI_CROSS_F32, config 4's DCN branch with fp32 output: 2 epilogue warps per quadrant at BN = 128 measured 354 ->
  // 320 us per launch; 4 warps of 32 columns each, 335)
  static constexpr int EPW = RING ? 3 : (ATTN ? 2 * ATT_GROUPS : (ATTN_TC ? 2 : (SPLIT ? (BN / 64 < EW ? BN / 64 : EW) : 1)));
  static constexpr int COLS_W = BN / EPW;           // columns per epilogue warp
  static constexpr int PRODUCER_B = 2 + 4 * EPW;
  static constexpr int PRODUCER_E = PRODUCER_B + 1;  // EIN producer (RING) / attention-MMA warps (ATTN_TC: +0, +1)
  static constexpr int NT = 32 * (PRODUCER_B + (RING ? 2 : (ATTN_TC ? 3 : 1)));
  static constexpr int OUT_BYTES = EpiTraits<EPI>::kSmemOut && !RING ? NSUB * SUB : 0;     // per buffer
  static constexpr int EIN_BYTES = EpiTraits<EPI>::kEin && !RING ? EpiTraits<EPI>::kEinTensors * NSUB * SUB : 0;  // per buf
  // EIN buffers: 2 (one per accumulator) by default; config 4's DCN U GEMM (fp32 output, 2-CTA 128-wide tiles) keeps
  // ONE, which leaves room for its split epilogue's fp32 staging and 4 operand ring stages (with 2 buffers and one
  // epilogue warp per quadrant it had 2 stages: 348-354 us; one buffer alone, 5 stages: no change; + the split
  // epilogue: 320 us) -- its B producer then issues a tile's x0 / x_l loads after the tile's weight k-blocks, once the
  // previous tile's epilogue has released the buffer
  // (MaskNet's EPI_MASK likewise: 2 -> 3 ring stages at BN = 128; c6 mask GEMM 30.3 -> 25.9 us, step 142 -> 137 us)
  static constexpr int EIN_NBUF = (EPI == EPI_CROSS_F32 || EPI == EPI_MASK) ? 1 : 2;
  // EPI_ATTN staging: Q | K | V of a tile's 128 tokens, bf16, row stride ATT_LD (padded: conflict-free ldmatrix).
  // (An unpadded XOR-swizzled layout freed a third ring stage but measured slower: 469 vs 381 us per layer.)
  static constexpr int ATT_LD = 72;
  static constexpr int ATT_BUF = 3 * BM * ATT_LD * 2;
  static constexpr int ATT_BYTES = ATTN ? ATT_GROUPS * ATT_BUF : (ATTN_TC ? 2 * 3 * SUB : 0);  // TC: [group][Q K V]
  // EPI_CROSS_F32 with a tmOut map: fp32 32 x 32 chunks staged per epilogue warp (double-buffered) and TMA-stored
  // (coalesced) instead of per-thread row stores
  static constexpr int F32_NBUF = CG == 2 ? 2 : 1;  // (single-CTA tiles: the ring needs the room)
  static constexpr int SLN_BUFS = 2;                 // EPI_SUM_LN: fp32 input chunks in flight per epilogue warp
  // shared-memory budget: 225 KB leaves room (2 x 1 KB reserved) for two co-resident gather CTAs of the next batch
  // (every kernel at 227 KB: c2 step 86.1 -> 95.2 us at two lanes, 97.2 -> 101.1 at one; c6 unchanged);
  // config 4's DCN U (fp32 output) and FFN2 + LN GEMMs take the whole 227 KB instead: one more operand ring stage
  // each (3 -> 4; SUM_LN with 2 input chunks per warp instead of 3): U 301 -> 284 us, FFN2 + LN 416 -> 377 us per
  // launch, c4 step -1.5-2% (its gather has the other GEMMs to hide under).  (MaskNet's mask GEMM at 227 KB: 26.2 ->
  // 23.8 us per launch but no faster c6 step -- its gather then loses those SMs.)
  // The 2-CTA (CG = 2) tiles -- config 4 only (pair_ens) -- likewise: FFN1 325 -> 315 us, the head's 16384 -> 2048
  // layer 440 -> 397 us (4 -> 5 stages).
  static constexpr int BUDGET = (EPI == EPI_CROSS_F32 || EPI == EPI_SUM_LN || CG == 2) ? 227 * 1024 : kSmemBudget;
  static constexpr int F32_BYTES = EPI == EPI_CROSS_F32 ? 4 * EPW * F32_NBUF * 32 * 32 * 4
                                  : (EPI == EPI_SUM_LN ? 4 * EPW * SLN_BUFS * 32 * 32 * 4 : 0);  // SUM_LN input ring
  static constexpr int EPI_BYTES =
      OUT_BUFS * OUT_BYTES + EIN_NBUF * EIN_BYTES + (RING ? RING_SLOTS * 2 * SUB : 0) + ATT_BYTES + F32_BYTES;
  static constexpr int BAR_BYTES = 512;
  // EPI_HEAD with a split epilogue: the EPW warps' partial dot products per row ([EPW][BM] fp32)
  static constexpr int Z_BYTES = EPI == EPI_HEAD ? EPW * BM * 4 : 0;
  static constexpr int STAGES_FIT = (BUDGET - 1024 - BAR_BYTES - EPI_BYTES - Z_BYTES) / STAGE;
#ifndef CVR_MAX_STAGES
#define CVR_MAX_STAGES 8
#endif
  static constexpr int STAGES = STAGES_FIT > CVR_MAX_STAGES ? CVR_MAX_STAGES : STAGES_FIT;
  // RING: a CTA's last tile (when it is not also its first) takes its epilogue inputs into the operand ring
  // instead of the slots -- the ring is free once that tile's MMAs have completed, long before the previous
  // tile's epilogue hands the slots back (sub-tile j: x0 in A stage j, x_l in B stage j)
  static constexpr bool RING_ALT = RING && NSUB <= STAGES && A_BYTES >= SUB && B_BYTES >= SUB;
  static constexpr int TMEM_COLS = 2 * BN <= 128 ? 128 : (2 * BN <= 256 ? 256 : 512);  // 2 accumulators, pow2 alloc
  static constexpr int SMEM = 1024 + STAGES * STAGE + EPI_BYTES + Z_BYTES + BAR_BYTES;
  static_assert(STAGES >= 2, "shared memory budget");
  // register cap: 65536 / NT (one CTA per SM), except the RING U GEMM (512 threads): 96 instead of 128 registers
  // (no spills) leaves 16K registers on each SM for two co-resident embedding CTAs of the next batch, which the
  // 128-register build locked out for the U GEMMs' whole duration -- c2 pipelined step 98.4 -> 97.1 us.  (The same
  // cap on the MLP GEMMs -- 80 or 64 registers -- measured 99.1 / 99.9 us, on the head -- 88 -- no change.)
  static constexpr int MAXREG_LB = (65536 / NT) > 255 ? 255 : (65536 / NT) & ~7;
  static constexpr int MAXREG = RING ? 96 : MAXREG_LB;
};

using namespace tile;

// CG = 2 (CTA pair, cluster of 2): a 256 x BN tile per pair with tcgen05.mma.cta_group::2 issued by the
// leader; each CTA loads its own 128 A rows and HALF of the B tile (BN/2 rows), so the bytes each SM must
// ingest per FLOP drop by (128 + BN/2)/(128 + BN); both CTAs' TMA bytes complete on the leader's full
// barrier, MMA completion is multicast to both CTAs, and each CTA runs the epilogue of its own 128 rows.
// Executor graphs (g.call): the row count M and the scores pointer are read from the per-call argument block in
// device memory; the grid is sized for max_batch and CTAs whose tiles lie beyond M find no work.
__device__ __forceinline__ void stamp(unsigned long long* dbg, int i) {
  if (dbg) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    dbg[blockIdx.x * 8 + i] = t;
  }
}

template <int BN, int EPI, int CG, int EW>
__global__ void __launch_bounds__(Cfg<BN, EPI, CG, EW>::NT, 1) __maxnreg__((Cfg<BN, EPI, CG, EW>::MAXREG))
    gemm_bf16_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const __grid_constant__ CUtensorMap tmOut, const __grid_constant__ CUtensorMap tmX0,
                     const __grid_constant__ CUtensorMap tmXl, const GemmArgs g) {
  using C = Cfg<BN, EPI, CG, EW>;
  using T = EpiTraits<EPI>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = sA + C::STAGES * C::A_BYTES;
  uint8_t* sOut = sB + C::STAGES * C::B_BYTES;         // [OUT_BUFS][NSUB][SUB]
  uint8_t* sEin = sOut + C::OUT_BUFS * C::OUT_BYTES;   // [2][x0 NSUB subs | x_l NSUB subs]
  // (ring slots / staging live in [sOut, sOut + EPI_BYTES); the head partials and the barriers follow them)
  float* zbuf = reinterpret_cast<float*>(sOut + C::EPI_BYTES);  // EPI_HEAD: [EPW][BM]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sOut + C::EPI_BYTES + C::Z_BYTES);
  uint64_t* full = bars;
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;   // [2] accumulator ready
  uint64_t* tempty = tfull + 2;          // [2] accumulator drained (4 epilogue warps)
  uint64_t* efull = tempty + 2;          // [3] epilogue input tiles (ring slots) landed
  uint64_t* eempty = efull + 3;          // [3] epilogue input tiles consumed (4 warps)
  uint64_t* sfull = eempty + 3;          // [4 warps][SLN_BUFS] EPI_SUM_LN fp32 input chunk landed
  uint64_t* abar = sfull + 4 * 3;        // [2 groups][4] EPI_ATTN_TC handshakes
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(abar + 8);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // executor graphs: this batch's row count (and scores pointer) from the per-call block, else the launch's
  const int M = g.call ? g.call->B * g.m_mult : g.M;
  const int N = g.N, K = g.K;
  constexpr int BMT = BM * CG;  // rows per tile (per CTA pair when CG = 2)
  const int rank = CG == 2 ? (int)ptx::cluster_ctarank() : 0;
  const bool leader = rank == 0;
  const int unit = CG == 2 ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
  const int n_units = CG == 2 ? (int)(gridDim.x >> 1) : (int)gridDim.x;
  const int n_tiles_n = N / BN;
  const int n_tiles = (M + BMT - 1) / BMT * n_tiles_n;
  auto tile_m = [&](int tile) { return tile / n_tiles_n; };
  auto tile_n = [&](int tile) { return tile % n_tiles_n; };
  float* const scores = g.call ? g.call->scores : g.scores;
  const int nk = K / BK;
  // tile walk: strided over the grid (n-fastest, so CTAs running together share the A row block in L2)
  const int t_begin = unit, t_end = n_tiles, t_step = n_units;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      ptx::mbar_init(&full[s], 2);  // one expect_tx arrival per producer stream
      ptx::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      ptx::mbar_init(&tfull[a], 1);
      ptx::mbar_init(&tempty[a], C::ATTN ? 4 * C::EPW / C::ATT_GROUPS : (C::ATTN_TC ? 4 : 4 * C::EPW * CG));
                                                                                           // (ATTN: of one group)
    }
    for (int e = 0; e < 3; ++e) {
      ptx::mbar_init(&efull[e], 1);
      ptx::mbar_init(&eempty[e], C::RING ? 4 : 4 * C::EPW);  // RING: one warp per quadrant and sub-tile slot
    }
    for (int i = 0; i < 8; ++i) ptx::mbar_init(&abar[i], 1);  // ATTN_TC: [group][qkv staged, S, P staged, O]
    for (int i = 0; i < 4 * 3; ++i) ptx::mbar_init(&sfull[i], 1);
    ptx::fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tmA);
    ptx::prefetch_tmap(&tmB);
    if (T::kSmemOut) ptx::prefetch_tmap(&tmOut);
    if (T::kEin) {
      ptx::prefetch_tmap(&tmX0);
      ptx::prefetch_tmap(&tmXl);
    }
  }
  if (warp == 1) {
    if constexpr (CG == 2) ptx::tmem_alloc_cg2(tmem_holder, C::TMEM_COLS);
    else ptx::tmem_alloc(tmem_holder, C::TMEM_COLS);
  }
  ptx::tc_fence_before();
  if constexpr (CG == 2) ptx::cluster_sync();  // peers' barriers exist before any remote arrive
  else __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  if (threadIdx.x == 0) stamp(g.dbg, 0);
  // B k-blocks of one tile (weights: never written by the previous kernel)
  auto issue_b = [&](int s, int kb, int n0) {
    if constexpr (CG == 2) {
      if (leader) ptx::mbar_arrive_expect_tx(&full[s], 2 * C::B_BYTES);
      ptx::tma_load_2d_cg2(sB + s * C::B_BYTES, &tmB, &full[s], kb * BK, n0 + rank * (BN / 2));
    } else {
      ptx::mbar_arrive_expect_tx(&full[s], C::B_BYTES);
      ptx::tma_load_2d(sB + s * C::B_BYTES, &tmB, &full[s], kb * BK, n0);
    }
  };
  // Weight prefetch: the first ring stages' B k-blocks are issued BEFORE griddepcontrol.wait, i.e. while the
  // previous kernel is still draining; only A (and the epilogue inputs) wait for it
  int npre = 0;
  if (!g.no_prefetch_b && warp == C::PRODUCER_B && lane == 0 && t_begin < t_end) {
    npre = nk < C::STAGES ? nk : C::STAGES;
    for (int kb = 0; kb < npre; ++kb) issue_b(kb, kb, tile_n(t_begin) * BN);
  }
  ptx::griddep_wait();  // inputs written by the previous kernel are visible from here on
  if (threadIdx.x == 0) stamp(g.dbg, 1);
  // Trigger the dependent launch now rather than at exit: its CTAs are then placed on each SM the moment
  // ours leaves it and run their prologue there, and only their griddepcontrol.wait (full completion +
  // flush of this grid) orders them after our results.  The grid is persistent (<= 1 CTA per SM, all
  // resident), so early dependents cannot starve our own CTAs.
  ptx::griddep_launch();

  if (warp == 0 || warp == C::PRODUCER_B) {
    // ================= TMA producers: warp 0 streams A (and the resident A blocks), warp 6 streams B and the
    // epilogue input tiles.  One issuing thread per operand stream: a single thread's TMA issue saturates
    // at ~69 B/clk/SM on B200 while two concurrent streams reach ~120 (scripts/micro/ingest_mix.cu).
    if (lane == 0) {
      const bool roleA = warp == 0;
      int gk = 0;     // global k-block counter (ring position)
      int it = 0;
      for (int tile = t_begin; tile < t_end; tile += t_step, ++it) {
        const int m0 = tile_m(tile) * BMT + rank * BM, n0 = tile_n(tile) * BN;
        // grouped GEMM (EPI_MASK over several MaskNet branches): N group g = n0 / group_n reads the K range
        // [g * K, (g + 1) * K) of A and the epilogue input at column n0 - g * group_n
        const int grp = (EPI == EPI_MASK && g.group_n > 0) ? n0 / g.group_n : 0;
        const int a_k0 = grp * K, e_n0 = n0 - grp * (EPI == EPI_MASK ? g.group_n : 0);
        auto issue_ein = [&]() {  // this tile's epilogue inputs (x0 / x_l tiles) into EIN buffer it % EIN_NBUF
          const int a = it % C::EIN_NBUF;
          if (it >= C::EIN_NBUF) ptx::mbar_wait(&eempty[a], ((it / C::EIN_NBUF) - 1) & 1);
          ptx::mbar_arrive_expect_tx(&efull[a], C::EIN_BYTES);
          uint8_t* base = sEin + a * C::EIN_BYTES;
#pragma unroll
          for (int j = 0; j < C::NSUB; ++j) {
            if constexpr (EPI == EPI_MASK) {
              ptx::tma_load_2d(base + j * C::SUB, &tmXl, &efull[a], e_n0 + j * 64, m0);
            } else {
              ptx::tma_load_2d(base + j * C::SUB, &tmX0, &efull[a], n0 + j * 64, m0);
              ptx::tma_load_2d(base + (C::NSUB + j) * C::SUB, &tmXl, &efull[a], n0 + j * 64, m0);
            }
          }
        };
        (void)issue_ein;
        if constexpr (T::kEin && !C::RING && C::EIN_NBUF == 2) {
          if (!roleA) issue_ein();
        }
        for (int kb = 0; kb < nk; ++kb, ++gk) {
          const int s = gk % C::STAGES;
          if (gk >= C::STAGES) ptx::mbar_wait(&empty[s], ((gk / C::STAGES) - 1) & 1);
          if (!roleA) {
            if (it > 0 || kb >= npre) issue_b(s, kb, n0);  // (first tile: the first npre were prefetched)
          } else if constexpr (CG == 2) {
            if (leader) ptx::mbar_arrive_expect_tx(&full[s], 2 * C::A_BYTES);
            ptx::tma_load_2d_cg2(sA + s * C::A_BYTES, &tmA, &full[s], kb * BK, m0);
          } else {
            ptx::mbar_arrive_expect_tx(&full[s], C::A_BYTES);
            ptx::tma_load_2d(sA + s * C::A_BYTES, &tmA, &full[s], a_k0 + kb * BK, m0);
          }
        }
        if constexpr (T::kEin && !C::RING && C::EIN_NBUF == 1) {
          if (!roleA) issue_ein();  // (single EIN buffer: after the tile's weight k-blocks, see Cfg::EIN_NBUF)
        }
      }
    }
  } else if (warp == C::PRODUCER_E && !C::ATTN_TC) {
    if constexpr (C::RING) {  // ================= EIN producer: (x0, x_l) 64-column sub-tile j -> slot j
      if (lane == 0) {
        int it = 0;
        for (int tile = t_begin; tile < t_end; tile += t_step, ++it) {
          const int m0 = tile_m(tile) * BMT + rank * BM, n0 = tile_n(tile) * BN;  // (CG = 2: this CTA's rows)
          const bool alt = C::RING_ALT && it >= 1 && tile + t_step >= t_end;
          // (tfull[a] is at most one phase behind here: tile it-2's epilogue released the slots, see below)
          if (alt) ptx::mbar_wait(&tfull[it & 1], (it >> 1) & 1);  // last tile's MMAs done: its ring is free
          for (int j = 0; j < C::NSUB; ++j) {
            uint8_t* x0d = alt ? sA + j * C::A_BYTES : sEin + j * 2 * C::SUB;
            uint8_t* xld = alt ? sB + j * C::B_BYTES : x0d + C::SUB;
            if (!alt && it >= 1) ptx::mbar_wait(&eempty[j], (it - 1) & 1);
            // alt: slot j's previous tile may still be landing -- its efull phase must complete before this
            // tile's expect_tx re-arms the barrier
            if (alt) ptx::mbar_wait(&efull[j], (it - 1) & 1);
            ptx::mbar_arrive_expect_tx(&efull[j], 2 * C::SUB);
            ptx::tma_load_2d(x0d, &tmX0, &efull[j], n0 + j * 64, m0);
            ptx::tma_load_2d(xld, &tmXl, &efull[j], n0 + j * 64, m0);
          }
        }
      }
    }
  } else if (C::ATTN_TC && warp >= C::PRODUCER_E) {
    if (lane == 0) {  // ================= attention MMAs of group grp's tiles (the tiles on accumulator grp)
      const int grp = warp - C::PRODUCER_E;
      const uint32_t sq = ptx::smem_u32(sOut + grp * 3 * C::SUB), sk = sq + C::SUB, sv = sq + 2 * C::SUB;
      const uint32_t acc = tmem + grp * BN;  // S in [0, 128), P (bf16 pairs) in [0, 64), O in [128, 192)
      constexpr uint32_t id_s = ptx::idesc_bf16_f32(128, 128), id_o = ptx::idesc_bf16_f32_bmn(128, 64);
      int j = 0;  // this group's tile count (barrier phase)
      for (int tile = t_begin + grp * t_step; tile < t_end; tile += 2 * t_step, ++j) {
        ptx::mbar_wait(&abar[grp * 4 + 0], j & 1);  // Q, K, V staged
        ptx::tc_fence_after();
#pragma unroll
        for (int k = 0; k < 4; ++k)  // S = Q K^T over dh = 64: both examples' 128 x 128 (cross blocks unused)
          ptx::umma_bf16_ss(acc, ptx::sdesc_kmajor_sw128(sq) + 2 * k, ptx::sdesc_kmajor_sw128(sk) + 2 * k, id_s, k);
        ptx::umma_commit(&abar[grp * 4 + 1]);
        ptx::mbar_wait(&abar[grp * 4 + 2], j & 1);  // P in TMEM (block diagonal over the 128 keys)
        ptx::tc_fence_after();
#pragma unroll
        for (int k = 0; k < 8; ++k)  // O = P V: A = P from TMEM (8 columns per 16 keys), V MN-major (2048 B per 16 keys)
          ptx::umma_bf16_ts(acc + 128, acc + 8 * k, ptx::sdesc_kmajor_sw128(sv) + 128 * k, id_o, k);
        ptx::umma_commit(&abar[grp * 4 + 3]);
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {  // ================= MMA issuer (the pair's leader when CG = 2)
      constexpr uint32_t idesc = ptx::idesc_bf16_f32(BMT, BN);
      int gk = 0, it = 0;
      for (int tile = t_begin; tile < t_end; tile += t_step, ++it) {
        const int a = it & 1;
        if (it >= 2) ptx::mbar_wait(&tempty[a], ((it >> 1) - 1) & 1);
        ptx::tc_fence_after();
        const uint32_t acc = tmem + a * BN;
        for (int kb = 0; kb < nk; ++kb, ++gk) {
          const int s = gk % C::STAGES;
          ptx::mbar_wait(&full[s], (gk / C::STAGES) & 1);
          if (gk == 0) stamp(g.dbg, 2);
          ptx::tc_fence_after();
          const uint64_t ad = ptx::sdesc_kmajor_sw128(ptx::smem_u32(sA + s * C::A_BYTES));
          const uint64_t bd = ptx::sdesc_kmajor_sw128(ptx::smem_u32(sB + s * C::B_BYTES));
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {  // K step 16 = 32 bytes = +2 in the 16-byte address field
            if constexpr (CG == 2) ptx::umma_bf16_ss_cg2(acc, ad + 2 * k, bd + 2 * k, idesc, (kb | k) != 0);
            else ptx::umma_bf16_ss(acc, ad + 2 * k, bd + 2 * k, idesc, (kb | k) != 0);
          }
          // frees the smem stage (in both CTAs of a pair) once these MMAs have read it
          if constexpr (CG == 2) ptx::umma_commit_cg2_mc(&empty[s]);
          else ptx::umma_commit(&empty[s]);
        }
        if constexpr (CG == 2) ptx::umma_commit_cg2_mc(&tfull[a]);  // accumulator a complete
        else ptx::umma_commit(&tfull[a]);
        stamp(g.dbg, 3);
      }
    }
  } else if (warp < C::PRODUCER_B) {  // ===== epilogue warps: TMEM quadrant q = warp % 4 -> rows 32q..32q+31
    const int q = warp & 3;
    const int part = (warp - 2) >> 2;  // RING: the 64-column sub-tile this warp finishes
    const int r = q * 32 + lane;  // row within the tile
    int it = 0, sln_k = 0;  // sln_k: EPI_SUM_LN fp32 input chunks consumed so far (ring position / parity)
    (void)part;
    (void)sln_k;
    for (int tile = t_begin; tile < t_end; tile += t_step, ++it) {
      const int m0 = tile_m(tile) * BMT + rank * BM, tn = tile_n(tile), n0 = tn * BN;
      const int m = m0 + r;
      const bool live = m < M;
      const int a = it & 1;
      if constexpr (C::ATTN) {
        if (a != (part >> 1)) continue;  // the other group's tile (its accumulator index)
      }
      if constexpr (C::ATTN_TC) {
        if (a != part) continue;  // the other group's tile
      }
      if constexpr (EPI == EPI_SUM_LN) {  // the tile's first fp32 input chunks (independent of the accumulator)
        if (lane == 0) {
          const int wq = warp - 2;
          ptx::fence_async_smem();  // this warp's reads of the ring (previous tile) before the TMA overwrites
          for (int i = 0; i < C::SLN_BUFS && 32 * i < BN; ++i) {
            const int b = (sln_k + i) % C::SLN_BUFS;
            ptx::mbar_arrive_expect_tx(&sfull[wq * 3 + b], 4096);
            ptx::tma_load_2d(sEin + C::EIN_NBUF * C::EIN_BYTES + (wq * C::SLN_BUFS + b) * 4096, &tmX0, &sfull[wq * 3 + b],
                             n0 + 32 * i, m0 + q * 32);
          }
        }
      }
      ptx::mbar_wait(&tfull[a], (it >> 1) & 1);
      if (it == 0 && warp == 2 && lane == 0) stamp(g.dbg, 4);
      ptx::tc_fence_after();
      const uint32_t trow = tmem + a * BN + ((uint32_t)(q * 32) << 16);
      const uint32_t out_base = ptx::smem_u32(sOut + (C::OUT_BUFS == 2 ? a : 0) * C::OUT_BYTES);
      const uint32_t ein_base = ptx::smem_u32(sEin + (it % C::EIN_NBUF) * C::EIN_BYTES);
      if constexpr (T::kEin && !C::RING) ptx::mbar_wait(&efull[it % C::EIN_NBUF], (it / C::EIN_NBUF) & 1);
      if constexpr (T::kSmemOut && !C::RING) {
        // the TMA store that last read this staging buffer must have finished reading it
        if (lane == 0) {
          if constexpr (C::OUT_BUFS == 2) ptx::bulk_wait_read<1>();
          else ptx::bulk_wait_read<0>();
        }
        __syncwarp();
      }
      float z = 0.f;
      if constexpr (C::RING) {
        // x_{l+1} = x0 * (acc + b) + x_l on sub-tile j = part, written over x_l in slot j and TMA-stored
        // from there; the slot is handed back once the store has read it
        const int j = part;
        const bool alt = C::RING_ALT && it >= 1 && tile + t_step >= t_end;  // inputs in the ring (see producer)
        ptx::mbar_wait(&efull[j], it & 1);
        uint8_t* xl_tile = alt ? sB + j * C::B_BYTES : sEin + j * 2 * C::SUB + C::SUB;
        const uint32_t x0b = ptx::smem_u32(alt ? sA + j * C::A_BYTES : sEin + j * 2 * C::SUB), xlb = ptx::smem_u32(xl_tile);
#pragma unroll
        for (int c = 0; c < 64; c += 32) {
          float v[32], x0v[32], xlv[32];
          ld32_tmem(trow + j * 64 + c, v);
          if (c == 32) {  // last TMEM read of this accumulator by this warp
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) {
              if constexpr (CG == 2) ptx::mbar_arrive_leader(&tempty[a]);
              else ptx::mbar_arrive(&tempty[a]);
            }
          }
          lds32_bf16(x0b, r, c >> 3, x0v);
          lds32_bf16(xlb, r, c >> 3, xlv);
          const float4* b4 = reinterpret_cast<const float4*>(g.bias + n0 + j * 64 + c);
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const float4 bb = __ldg(b4 + u);
            v[4 * u] = x0v[4 * u] * (v[4 * u] + bb.x) + xlv[4 * u];
            v[4 * u + 1] = x0v[4 * u + 1] * (v[4 * u + 1] + bb.y) + xlv[4 * u + 1];
            v[4 * u + 2] = x0v[4 * u + 2] * (v[4 * u + 2] + bb.z) + xlv[4 * u + 2];
            v[4 * u + 3] = x0v[4 * u + 3] * (v[4 * u + 3] + bb.w) + xlv[4 * u + 3];
          }
          sts32_bf16(xlb, r, c >> 3, v);
        }
        ptx::fence_async_smem();
        __syncwarp();
        if (lane == 0) {
          ptx::tma_store_2d(&tmOut, xl_tile + q * 32 * 128, n0 + j * 64, m0 + q * 32);
          ptx::bulk_commit();
          ptx::bulk_wait_read<0>();
          ptx::mbar_arrive(&eempty[j]);
        }
        __syncwarp();
      } else if constexpr (C::ATTN_TC) {
        // ---- fused QKV projection + attention on tcgen05 (config 4, SURVEY.md §8(a) S5', A20): rows [m0, m0 + 128) =
        // two examples' 64 tokens, columns [q_h | k_h | v_h] of head h = tn.  Same roundings as EPI_ATTN / mha64: q, k,
        // v + bias rounded to bf16, S = Q K^T fp32, softmax(S / 8) fp32 (exact scale), P rounded to bf16, O fp32 -> bf16.
        const int grp = a;  // this warp's group owns the tiles on accumulator `grp`
        uint64_t* ab = abar + grp * 4;
        const int j = it >> 1;  // the group's tile count (barrier phase)
        const uint32_t sq = ptx::smem_u32(sOut + grp * 3 * C::SUB);
        const uint32_t acc = tmem + a * BN + ((uint32_t)(q * 32) << 16);
        const bool lead = q == 0 && lane == 0;
        // (0) the previous O store of this group has read the staging (Q doubles as O)
        if (lead) ptx::bulk_wait_read<0>();
        ptx::named_bar_sync(1 + grp, 32 * 4);
        // (1) accumulator + bias -> bf16 Q | K | V rows
#pragma unroll 1
        for (int c = 0; c < 192; c += 32) {
          float v[32];
          ld32_tmem(trow + c, v);
          const float4* b4 = reinterpret_cast<const float4*>(g.bias + n0 + c);
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const float4 bb = __ldg(b4 + u);
            v[4 * u] += bb.x;
            v[4 * u + 1] += bb.y;
            v[4 * u + 2] += bb.z;
            v[4 * u + 3] += bb.w;
          }
          sts32_bf16(sq + (c >> 6) * C::SUB, r, (c & 63) >> 3, v);
        }
        ptx::fence_async_smem();  // generic-proxy staging writes -> visible to the tensor core's reads
        ptx::tc_fence_before();
        ptx::named_bar_sync(1 + grp, 32 * 4);
        if (lead) ptx::mbar_arrive(&ab[0]);
        // (2) softmax of this row over its example's 64 keys (columns [64 e, 64 e + 64) of S); P (bf16) back into TMEM
        // columns [0, 64) as pairs (keys 2i, 2i + 1 in column i), the other example's 32 columns zero
        ptx::mbar_wait(&ab[1], j & 1);
        ptx::tc_fence_after();
        {
          const int e = r >> 6;
          float s0[32], s1[32];
          ld32_tmem(acc + 64 * e, s0);
          ld32_tmem(acc + 64 * e + 32, s1);
          float mx = -INFINITY;
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            s0[i] *= 0.125f;
            s1[i] *= 0.125f;
            mx = fmaxf(mx, fmaxf(s0[i], s1[i]));
          }
          float sum = 0.f;
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            s0[i] = expf(s0[i] - mx);
            s1[i] = expf(s1[i] - mx);
            sum += s0[i];
          }
#pragma unroll
          for (int i = 0; i < 32; ++i) sum += s1[i];
          const float inv = 1.f / sum;
          uint32_t pk[16], z[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            pk[i] = ptx::pack_bf16(s0[2 * i] * inv, s0[2 * i + 1] * inv);
            z[i] = 0u;
          }
          ptx::tmem_st_32x32b_x16(acc + 32 * e, pk);
#pragma unroll
          for (int i = 0; i < 16; ++i) pk[i] = ptx::pack_bf16(s1[2 * i] * inv, s1[2 * i + 1] * inv);
          ptx::tmem_st_32x32b_x16(acc + 32 * e + 16, pk);
          ptx::tmem_st_32x32b_x16(acc + 32 * (1 - e), z);
          ptx::tmem_st_32x32b_x16(acc + 32 * (1 - e) + 16, z);
          ptx::tmem_wait_st();
        }
        ptx::tc_fence_before();
        ptx::named_bar_sync(1 + grp, 32 * 4);
        if (lead) ptx::mbar_arrive(&ab[2]);
        // (3) O rows -> bf16 staging (over Q) -> one TMA store of the 128 x 64 box at cat[m0.., 64 h]
        ptx::mbar_wait(&ab[3], j & 1);
        ptx::tc_fence_after();
#pragma unroll
        for (int c = 0; c < 64; c += 32) {
          float o[32];
          ld32_tmem(acc + 128 + c, o);
          sts32_bf16(sq, r, c >> 3, o);
        }
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&tempty[a]);  // accumulator a (QKV, S, P, O columns) free for its next tile
        ptx::fence_async_smem();
        ptx::named_bar_sync(1 + grp, 32 * 4);
        if (lead) {
          ptx::tma_store_2d(&tmOut, sOut + grp * 3 * C::SUB, tn * 64, m0);
          ptx::bulk_commit();
        }
      } else if constexpr (C::ATTN) {
        // ---- fused QKV projection + attention (config 4, SURVEY.md §8(a) S5', A20): this tile is rows [m0, m0+128)
        // = two examples' 64 tokens, columns [q_h | k_h | v_h] of head h = tn (weights repacked head-major at load)
        const int grp = part >> 1, gpart = part & 1;  // group = accumulator of its tiles; 2 warps per quadrant
        __nv_bfloat16* qs = reinterpret_cast<__nv_bfloat16*>(sOut + grp * C::ATT_BUF);  // [3][128][ATT_LD]
        constexpr int LDA = C::ATT_LD;
        // (1) accumulator + bias -> bf16 Q / K / V rows (the QKV GEMM's EPI_BIAS rounding); warp (q, part) converts
        //     its TMEM quadrant's 32 rows, columns [96 part, 96 part + 96)
#pragma unroll 1
        for (int cc = 0; cc < 3; ++cc) {
          const int c = gpart * 96 + cc * 32;
          float v[32];
          ld32_tmem(trow + c, v);
          const float4* b4 = reinterpret_cast<const float4*>(g.bias + n0 + c);
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const float4 bb = __ldg(b4 + u);
            v[4 * u] += bb.x;
            v[4 * u + 1] += bb.y;
            v[4 * u + 2] += bb.z;
            v[4 * u + 3] += bb.w;
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            uint4 o;
            o.x = ptx::pack_bf16(v[8 * u], v[8 * u + 1]);
            o.y = ptx::pack_bf16(v[8 * u + 2], v[8 * u + 3]);
            o.z = ptx::pack_bf16(v[8 * u + 4], v[8 * u + 5]);
            o.w = ptx::pack_bf16(v[8 * u + 6], v[8 * u + 7]);
            *reinterpret_cast<uint4*>(qs + ((c >> 6) * BM + r) * LDA + (c & 63) + 8 * u) = o;
          }
        }
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&tempty[a]);  // the accumulator is free for the tile after next
        ptx::named_bar_sync(1 + grp, 32 * 8);     // every token's Q / K / V is staged
        // (2) attention (cvr_attn.cuh, the mha64 core): warp ew = 4 gpart + q -> example ew / 4, query rows 16 (ew % 4)
        const int ew = gpart * 4 + q, ex = ew >> 2, r0 = (ew & 3) * 16;
        __nv_bfloat16* Qs = qs + (ex * 64) * LDA;
        attn::rows16<LDA>(Qs, qs + (BM + ex * 64) * LDA, qs + (2 * BM + ex * 64) * LDA, r0, lane);
        __syncwarp();
        // (3) O rows -> out (16 rows x 128 B, coalesced 16-byte chunks)
#pragma unroll
        for (int p = 0; p < 4; ++p) {
          const int row = p * 4 + (lane >> 3), ch = lane & 7, tok = m0 + ex * 64 + r0 + row;
          if (tok < M)
            *reinterpret_cast<uint4*>(g.out_bf16 + (int64_t)tok * g.ld_x + tn * 64 + ch * 8) =
                *reinterpret_cast<const uint4*>(Qs + (r0 + row) * LDA + ch * 8);
        }
        ptx::named_bar_sync(1 + grp, 32 * 8);  // the group's staging buffer is free for its next tile
      } else if constexpr (EPI == EPI_SUM_LN) {
        // pass 1: y = acc + b + in, written back into TMEM; row sum.  The fp32 input (this warp's 32 rows x 32-column
        // chunks) arrives by TMA into a per-warp ring of SLN_BUFS swizzled 4 KB buffers, the first chunks issued
        // before the accumulator is ready (per-lane row reads touched 32 lines per instruction and exposed the
        // memory latency of every chunk: 1.5x slower kernel)
        float sum = 0.f;
        const int wq = warp - 2;  // (EPW = 1: one warp per quadrant)
#pragma unroll 1
        for (int c = 0; c < BN; c += 32) {
          const int k = sln_k + (c >> 5), b = k % C::SLN_BUFS;
          float v[32], x[32];
          ld32_tmem(trow + c, v);
          ptx::mbar_wait(&sfull[wq * 3 + b], (k / C::SLN_BUFS) & 1);
          const uint32_t xt = ptx::smem_u32(sEin + C::EIN_NBUF * C::EIN_BYTES + (wq * C::SLN_BUFS + b) * 4096);
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const uint4 w4 = lds128(xt + lane * 128 + ((u ^ (lane & 7)) << 4));
            x[4 * u] = __uint_as_float(w4.x);
            x[4 * u + 1] = __uint_as_float(w4.y);
            x[4 * u + 2] = __uint_as_float(w4.z);
            x[4 * u + 3] = __uint_as_float(w4.w);
          }
          __syncwarp();
          if (lane == 0 && c + 32 * C::SLN_BUFS < BN) {  // refill this buffer with chunk c + SLN_BUFS of the tile
            ptx::fence_async_smem();
            ptx::mbar_arrive_expect_tx(&sfull[wq * 3 + b], 4096);
            ptx::tma_load_2d(sEin + C::EIN_NBUF * C::EIN_BYTES + (wq * C::SLN_BUFS + b) * 4096, &tmX0, &sfull[wq * 3 + b],
                             n0 + c + 32 * C::SLN_BUFS, m0 + q * 32);
          }
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            v[j] = v[j] + __ldg(g.bias + n0 + c + j) + (live ? x[j] : 0.f);
            sum += v[j];
          }
          st32_tmem(trow + c, v);
        }
        sln_k += BN / 32;
        ptx::tmem_wait_st();
        const float mean = sum / (float)BN;
        float var = 0.f;  // pass 2: centred second moment (biased variance, A20)
#pragma unroll 1
        for (int c = 0; c < BN; c += 32) {
          float v[32];
          ld32_tmem(trow + c, v);
#pragma unroll
          for (int j = 0; j < 32; ++j) var = fmaf(v[j] - mean, v[j] - mean, var);
        }
        const float rstd = 1.f / sqrtf(var / (float)BN + 1e-5f);
#pragma unroll 1
        for (int c = 0; c < BN; c += 32) {  // pass 3: normalise, affine, bf16
          float v[32];
          ld32_tmem(trow + c, v);
#pragma unroll
          for (int j = 0; j < 32; ++j)
            v[j] = (v[j] - mean) * rstd * __ldg(g.gamma + n0 + c + j) + __ldg(g.beta + n0 + c + j);
          sts32_bf16(out_base + (c >> 6) * C::SUB, r, (c & 63) >> 3, v);
        }
      } else {
#pragma unroll 1
        for (int c = part * C::COLS_W; c < (part + 1) * C::COLS_W; c += 32) {
          float v[32];
          ld32_tmem(trow + c, v);
          const int n = n0 + c;
          if constexpr (T::kBias) {  // bias / head weights: fp32, 16-byte aligned (workspace slots; cvr.h)
            const float4* b4 = reinterpret_cast<const float4*>(g.bias + n);
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              const float4 bb = __ldg(b4 + u);
              v[4 * u] += bb.x;
              v[4 * u + 1] += bb.y;
              v[4 * u + 2] += bb.z;
              v[4 * u + 3] += bb.w;
            }
          }
          if constexpr (EPI == EPI_HEAD || EPI == EPI_HEAD_PARTIAL) {
            const float4* h4 = reinterpret_cast<const float4*>(g.head_w + n);
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              const float4 hw = __ldg(h4 + u);
              z = fmaf(fmaxf(v[4 * u], 0.f), hw.x, z);
              z = fmaf(fmaxf(v[4 * u + 1], 0.f), hw.y, z);
              z = fmaf(fmaxf(v[4 * u + 2], 0.f), hw.z, z);
              z = fmaf(fmaxf(v[4 * u + 3], 0.f), hw.w, z);
            }
          } else if constexpr (EPI == EPI_BIAS_ADD_F32) {
            if (live) {
              float x[32];
              ld32_f32(g.in_f32 + (int64_t)m * g.ld_in + n, x);
#pragma unroll
              for (int j = 0; j < 32; ++j) v[j] += x[j];
              st32_f32(g.out_f32 + (int64_t)m * g.ld_f32 + n, v);
            }
          } else {
            if constexpr (EPI == EPI_BIAS_RELU) {
#pragma unroll
              for (int j = 0; j < 32; ++j) v[j] = fmaxf(v[j], 0.f);
            }
            if constexpr (EPI == EPI_MASK) {
              float xlv[32];
              lds32_bf16(ein_base + (c >> 6) * C::SUB, r, (c & 63) >> 3, xlv);
#pragma unroll
              for (int j = 0; j < 32; ++j) v[j] = v[j] * xlv[j];
            } else if constexpr (T::kEin) {
              float x0v[32], xlv[32];
              lds32_bf16(ein_base + (c >> 6) * C::SUB, r, (c & 63) >> 3, x0v);
              lds32_bf16(ein_base + (C::NSUB + (c >> 6)) * C::SUB, r, (c & 63) >> 3, xlv);
#pragma unroll
              for (int j = 0; j < 32; ++j) v[j] = x0v[j] * v[j] + xlv[j];
            }
            if constexpr (EPI == EPI_CROSS_F32) {
              if (g.tmOut) {  // (the launch passed a store map: use its kernel-parameter copy)
                // stage this warp's 32 rows x 32 columns (swizzled 16-byte chunks), one TMA store per chunk
                const int buf = (c >> 5) % C::F32_NBUF;
                uint8_t* sb = sEin + C::EIN_NBUF * C::EIN_BYTES + ((warp - 2) * C::F32_NBUF + buf) * 4096;
                if (lane == 0) ptx::bulk_wait_read<C::F32_NBUF - 1>();  // the last store from this buffer read it
                __syncwarp();
                const uint32_t sbu = ptx::smem_u32(sb);
#pragma unroll
                for (int u = 0; u < 8; ++u)
                  sts128(sbu + lane * 128 + ((u ^ (lane & 7)) << 4),
                         make_uint4(__float_as_uint(v[4 * u]), __float_as_uint(v[4 * u + 1]),
                                    __float_as_uint(v[4 * u + 2]), __float_as_uint(v[4 * u + 3])));
                ptx::fence_async_smem();
                __syncwarp();
                if (lane == 0) {
                  ptx::tma_store_2d(&tmOut, sb, n, m0 + q * 32);
                  ptx::bulk_commit();
                }
              } else if (live) {
                st32_f32(g.out_f32 + (int64_t)m * g.ld_f32 + n, v);
              }
            } else {
              sts32_bf16(out_base + (c >> 6) * C::SUB, r, (c & 63) >> 3, v);
            }
          }
        }
      }
      // accumulator (and epilogue inputs) consumed: hand them back (RING / ATTN warps did so themselves)
      if constexpr (!C::RING && !C::ATTN && !C::ATTN_TC) {
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if constexpr (CG == 2) ptx::mbar_arrive_leader(&tempty[a]);
          else ptx::mbar_arrive(&tempty[a]);
          if constexpr (T::kEin) ptx::mbar_arrive(&eempty[it % C::EIN_NBUF]);
        }
      }
      if constexpr (EPI == EPI_HEAD && C::EPW > 1) {
        // split epilogue: the quadrant's EPW warps hand their partial dot products to part 0, which sums them in
        // column order from 0 (as the cluster head sums its CTAs' partials in rank order: same result)
        zbuf[part * BM + r] = z;
        ptx::named_bar_sync(1 + q, 32 * C::EPW);
        if (part == 0) {
          float zs = 0.f;
#pragma unroll
          for (int j = 0; j < C::EPW; ++j) zs += zbuf[j * BM + r];
          if (live) scores[m] = sigmoid_f32(zs + g.head_b);
        }
        ptx::named_bar_sync(1 + q, 32 * C::EPW);  // zbuf free for the next tile
      } else if constexpr (EPI == EPI_HEAD) {
        if (live) scores[m] = sigmoid_f32(z + g.head_b);
      } else if constexpr (EPI == EPI_HEAD_PARTIAL) {
        if (live) g.partial[(int64_t)m * n_tiles_n + tn] = z;
      } else if constexpr (T::kSmemOut && !C::RING) {
        ptx::fence_async_smem();
        __syncwarp();
        if (lane == 0) {
          const uint8_t* ob = sOut + (C::OUT_BUFS == 2 ? a : 0) * C::OUT_BYTES;
#pragma unroll
          for (int j = 0; j < C::NSUB; ++j)
            if (j * 64 >= part * C::COLS_W && j * 64 < (part + 1) * C::COLS_W)
              ptx::tma_store_2d(&tmOut, ob + j * C::SUB + q * 32 * 128, n0 + j * 64, m0 + q * 32);
          ptx::bulk_commit();
        }
      }
    }
    if constexpr (T::kSmemOut || C::RING || EPI == EPI_CROSS_F32 || C::ATTN_TC) {
      if (lane == 0) ptx::bulk_wait<0>();
    }
    if (warp == 2 && lane == 0) stamp(g.dbg, 5);
  }
  ptx::tc_fence_before();
  // CG = 2: both CTAs are done with the pair's TMEM
  if constexpr (CG == 2) ptx::cluster_sync();
  else __syncthreads();
  if (threadIdx.x == 0) stamp(g.dbg, 6);
  if (warp == 1) {
    if constexpr (CG == 2) ptx::tmem_dealloc_cg2(tmem, C::TMEM_COLS);
    else ptx::tmem_dealloc(tmem, C::TMEM_COLS);
  }
}

template <int BN, int EPI, int CG = 1, int EW = 4>
cudaError_t launch_t(const GemmArgs& g, cudaStream_t s) {
  using C = Cfg<BN, EPI, CG, EW>;
  auto kern = gemm_bf16_kernel<BN, EPI, CG, EW>;
  static bool attr_done = false;
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return e;
    attr_done = true;
  }
  // (executor graphs: g.M is max_batch * m_mult here, the kernel reads the batch's M from g.call)
  const int m_blocks = (g.M + BM * CG - 1) / (BM * CG);
  const int n_tiles = m_blocks * (g.N / BN);
  const int max_units = g.num_sms / CG;
  const int grid = (n_tiles < max_units ? n_tiles : max_units) * CG;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(C::NT);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = g.pdl ? 1 : 0;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = CG;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = CG > 1 ? 2 : 1;
  const CUtensorMap* dummy = g.tmA;
  return cudaLaunchKernelEx(&cfg, kern, *g.tmA, *g.tmB, *(g.tmOut ? g.tmOut : dummy), *(g.tmX0 ? g.tmX0 : dummy),
                            *(g.tmXl ? g.tmXl : dummy), g);
}

}  // namespace

// instantiated (BN, epilogue) pairs: the shared-memory budget allows the double-buffered
// x0/x_l/out tiles of EPI_CROSS only at BN = 64, and staged bf16 outputs up to BN = 128.
cudaError_t launch_gemm_bf16(const GemmArgs& g, cudaStream_t s) {
  if (g.M <= 0) return cudaSuccess;
  const bool full_row = g.epi == EPI_HEAD || g.epi == EPI_SUM_LN;
  if (g.K % BK || g.N % g.BN || (full_row && g.BN != g.N)) return cudaErrorInvalidValue;
  if (g.call && g.m_mult <= 0) return cudaErrorInvalidValue;
  if ((g.epi == EPI_STORE || g.epi == EPI_BIAS_RELU || g.epi == EPI_CROSS || g.epi == EPI_BIAS ||
       g.epi == EPI_SUM_LN) && !g.tmOut)
    return cudaErrorInvalidValue;
  if ((g.epi == EPI_CROSS || g.epi == EPI_CROSS_F32) && (!g.tmX0 || !g.tmXl)) return cudaErrorInvalidValue;
  if (g.epi == EPI_SUM_LN && !g.tmX0) return cudaErrorInvalidValue;  // the fp32 input's TMA load map
  if (g.epi == EPI_MASK && (!g.tmXl || !g.tmOut)) return cudaErrorInvalidValue;
  // one epilogue warp per quadrant when every CTA runs several tiles (see Cfg::EPW)
  if (g.epw1 && g.cta_pair && (g.epi == EPI_STORE || g.epi == EPI_BIAS_RELU || g.epi == EPI_BIAS)) {
#define CVR_E1P(BN_, EPI_) \
    if (g.BN == BN_ && g.epi == EPI_) return launch_t<BN_, EPI_, 2, 1>(g, s);
    CVR_E1P(128, EPI_STORE)
    CVR_E1P(256, EPI_STORE)
    CVR_E1P(128, EPI_BIAS_RELU)
    CVR_E1P(256, EPI_BIAS_RELU)
    CVR_E1P(128, EPI_BIAS)
    CVR_E1P(256, EPI_BIAS)
#undef CVR_E1P
  }
  if (g.epw1 && !g.cta_pair && (g.epi == EPI_STORE || g.epi == EPI_BIAS_RELU || g.epi == EPI_BIAS)) {
#define CVR_E1(BN_, EPI_) \
    if (g.BN == BN_ && g.epi == EPI_) return launch_t<BN_, EPI_, 1, 1>(g, s);
    CVR_E1(128, EPI_STORE)
    CVR_E1(192, EPI_STORE)
    CVR_E1(256, EPI_STORE)
    CVR_E1(128, EPI_BIAS_RELU)
    CVR_E1(256, EPI_BIAS_RELU)
    CVR_E1(128, EPI_BIAS)
    CVR_E1(256, EPI_BIAS)
#undef CVR_E1
  }
  if (g.epi == EPI_ATTN) {
    if (g.BN != 192 || g.N % 192 || g.cta_pair || !g.out_bf16 || !g.bias || g.ld_x % 8) return cudaErrorInvalidValue;
    return launch_t<192, EPI_ATTN>(g, s);
  }
  if (g.epi == EPI_ATTN_TC) {
    if (g.BN != 192 || g.N % 192 || g.cta_pair || !g.tmOut || !g.bias) return cudaErrorInvalidValue;
    return launch_t<192, EPI_ATTN_TC>(g, s);
  }
#define CVR_CASE(BN_, EPI_) \
  if (g.BN == BN_ && g.epi == EPI_) return g.cta_pair ? launch_t<BN_, EPI_, 2>(g, s) : launch_t<BN_, EPI_>(g, s);
  CVR_CASE(64, EPI_STORE)
  CVR_CASE(128, EPI_STORE)
  CVR_CASE(256, EPI_STORE)
  CVR_CASE(192, EPI_STORE)
  CVR_CASE(256, EPI_BIAS_RELU)
  CVR_CASE(64, EPI_BIAS_RELU)
  CVR_CASE(128, EPI_BIAS_RELU)
  CVR_CASE(64, EPI_CROSS)
  if (g.BN == 192 && g.epi == EPI_CROSS && !g.cta_pair) return launch_t<192, EPI_CROSS>(g, s);
  CVR_CASE(64, EPI_HEAD)
  CVR_CASE(128, EPI_HEAD)
  CVR_CASE(256, EPI_HEAD)
  CVR_CASE(128, EPI_BIAS)
  CVR_CASE(256, EPI_BIAS)
  CVR_CASE(64, EPI_CROSS_F32)
  CVR_CASE(128, EPI_CROSS_F32)
  CVR_CASE(64, EPI_BIAS_ADD_F32)
  CVR_CASE(128, EPI_BIAS_ADD_F32)
  CVR_CASE(256, EPI_SUM_LN)
  CVR_CASE(256, EPI_HEAD_PARTIAL)
  CVR_CASE(64, EPI_MASK)
  CVR_CASE(128, EPI_MASK)
#undef CVR_CASE
  return cudaErrorInvalidValue;
}

int encode_tmap_f32_store(CUtensorMap* tm, const void* ptr, int64_t rows, int64_t cols, int64_t ld, const char** err) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn) {
      *err = "cuTensorMapEncodeTiled entry point unavailable";
      return -1;
    }
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  cuuint64_t gdim[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t gstride[1] = {(cuuint64_t)ld * 4};
  cuuint32_t box[2] = {32, 32};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(ptr), gdim, gstride, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    *err = "cuTensorMapEncodeTiled (fp32) failed";
    return -1;
  }
  return 0;
}

int encode_tmap_bf16(CUtensorMap* tm, const void* ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows,
                     const char** err) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn) {
      *err = "cuTensorMapEncodeTiled entry point unavailable";
      return -1;
    }
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  cuuint64_t gdim[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t gstride[1] = {(cuuint64_t)ld * 2};
  cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode(tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), gdim, gstride, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    *err = "cuTensorMapEncodeTiled failed";
    return -1;
  }
  return 0;
}

}  // namespace cvr
