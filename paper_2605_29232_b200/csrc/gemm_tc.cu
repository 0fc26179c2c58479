// gemm_tc.cu -- K4: bf16 GEMM on the 5th-generation tensor cores (tcgen05 + TMEM + TMA) with the
// dense stage's elementwise work fused into the epilogue:
//
//   EPI_STORE      C = A B^T                         t = x_l V_l^T
//   EPI_CROSS      C = x0 * (A B^T + b) + x_l        x_{l+1} = x0 * (U_l t + b_l) + x_l
//                                                    (PAPER.md:225 low-rank DCNv2; A9 bias)
//   EPI_BIAS_RELU  C = ReLU(A B^T + b)               MLP tower
//   EPI_HEAD       s = sigmoid(ReLU(A B^T + b) . m + c)   last MLP layer + head, h never stored
//                                                    (BASELINE.json north star)
//
// A [M, K] and B [N, K] are bf16, K-major, moved by TMA into 128-byte-swizzled shared memory
// (BK = 64 elements = one swizzle atom).  One CTA computes a BM=128 x BN tile: warp 0 is the
// TMA producer, warp 1 allocates TMEM and one elected lane issues tcgen05.mma (M=128, N=BN,
// K=16) into a 128-lane x BN-column fp32 TMEM accumulator, warps 2-5 are the epilogue (each
// reads its 32-lane TMEM quadrant with tcgen05.ld, one row per thread).  A STAGES-deep
// full/empty mbarrier ring overlaps TMA with MMA.  No split-K: every row's result depends only
// on that row, in a fixed K order, so scores are batch-invariant.
#include <cudaTypedefs.h>
#include <cuda_bf16.h>

#include "cvr_kernels.cuh"
#include "cvr_ptx.cuh"

namespace cvr {
namespace {

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int kThreads = 192;

template <int BN>
struct Cfg {
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int STAGES = BN == 256 ? 4 : (BN == 128 ? 6 : 8);
  static constexpr int TMEM_COLS = BN;  // 64 / 128 / 256: powers of two >= 32
  static constexpr int SMEM = STAGES * STAGE + 1024 + 256;
};

__device__ __forceinline__ float sigmoid_f32(float z) {
  if (z >= 0.f) return 1.f / (1.f + expf(-z));
  const float e = expf(z);
  return e / (1.f + e);
}

__device__ __forceinline__ void load16_bf16(const __nv_bfloat16* p, float (&v)[16]) {
  const uint4 a = *reinterpret_cast<const uint4*>(p);
  const uint4 b = *reinterpret_cast<const uint4*>(p + 8);
  const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    v[2 * i] = ptx::bf16_lo(w[i]);
    v[2 * i + 1] = ptx::bf16_hi(w[i]);
  }
}
__device__ __forceinline__ void store16_bf16(__nv_bfloat16* p, const float (&v)[16]) {
  uint4 a, b;
  a.x = ptx::pack_bf16(v[0], v[1]);
  a.y = ptx::pack_bf16(v[2], v[3]);
  a.z = ptx::pack_bf16(v[4], v[5]);
  a.w = ptx::pack_bf16(v[6], v[7]);
  b.x = ptx::pack_bf16(v[8], v[9]);
  b.y = ptx::pack_bf16(v[10], v[11]);
  b.z = ptx::pack_bf16(v[12], v[13]);
  b.w = ptx::pack_bf16(v[14], v[15]);
  *reinterpret_cast<uint4*>(p) = a;
  *reinterpret_cast<uint4*>(p + 8) = b;
}

template <int BN, int EPI>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_bf16_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const EpiParams p, int M, int K) {
  using C = Cfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::STAGES * C::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE);
  uint64_t* empty = full + C::STAGES;
  uint64_t* done = empty + C::STAGES;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(done + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n0 = blockIdx.x * BN, m0 = blockIdx.y * BM;
  const int nk = K / BK;

  if (threadIdx.x == 0) {
#pragma unroll
    for (int s = 0; s < C::STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    ptx::mbar_init(done, 1);
    ptx::fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tmA);
    ptx::prefetch_tmap(&tmB);
  }
  if (warp == 1) ptx::tmem_alloc(tmem_holder, C::TMEM_COLS);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_holder;

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % C::STAGES;
        if (kb >= C::STAGES) ptx::mbar_wait(&empty[s], ((kb / C::STAGES) - 1) & 1);
        ptx::mbar_arrive_expect_tx(&full[s], C::STAGE);
        ptx::tma_load_2d(sA + s * C::A_BYTES, &tmA, &full[s], kb * BK, m0);
        ptx::tma_load_2d(sB + s * C::B_BYTES, &tmB, &full[s], kb * BK, n0);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer (single thread)
      constexpr uint32_t idesc = ptx::idesc_bf16_f32(BM, BN);
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % C::STAGES;
        ptx::mbar_wait(&full[s], (kb / C::STAGES) & 1);
        ptx::tc_fence_after();
        const uint64_t ad = ptx::sdesc_kmajor_sw128(ptx::smem_u32(sA + s * C::A_BYTES));
        const uint64_t bd = ptx::sdesc_kmajor_sw128(ptx::smem_u32(sB + s * C::B_BYTES));
#pragma unroll
        for (int k = 0; k < BK / 16; ++k)  // K step 16 = 32 bytes = +2 in the 16-byte address field
          ptx::umma_bf16_ss(tmem, ad + 2 * k, bd + 2 * k, idesc, (kb | k) != 0);
        ptx::umma_commit(&empty[s]);  // frees the smem stage once these MMAs have read it
      }
      ptx::umma_commit(done);  // accumulator complete
    }
    __syncwarp();
  } else {  // ---- epilogue warps 2..5: TMEM quadrant q = warp % 4 holds rows 32q .. 32q+31
    ptx::mbar_wait(done, 0);
    ptx::tc_fence_after();
    const int q = warp & 3;
    const int m = m0 + q * 32 + lane;
    const bool live = m < M;
    const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16);
    float z = 0.f;
#pragma unroll 1
    for (int c = 0; c < BN; c += 16) {
      uint32_t r[16];
      ptx::tmem_ld_32x32b_x16(trow + c, r);
      ptx::tmem_wait_ld();
      float v[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(r[j]);
      const int n = n0 + c;
      if constexpr (EPI == EPI_STORE) {
        if (live) store16_bf16(reinterpret_cast<__nv_bfloat16*>(p.out) + (int64_t)m * p.ldo + n, v);
      } else if constexpr (EPI == EPI_BIAS_RELU) {
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = fmaxf(v[j] + __ldg(p.bias + n + j), 0.f);
        if (live) store16_bf16(reinterpret_cast<__nv_bfloat16*>(p.out) + (int64_t)m * p.ldo + n, v);
      } else if constexpr (EPI == EPI_CROSS) {
        if (live) {
          float x0v[16], xlv[16];
          load16_bf16(p.x0 + (int64_t)m * p.ld_x0 + n, x0v);
          load16_bf16(p.xl + (int64_t)m * p.ld_xl + n, xlv);
#pragma unroll
          for (int j = 0; j < 16; ++j) v[j] = x0v[j] * (v[j] + __ldg(p.bias + n + j)) + xlv[j];
          store16_bf16(reinterpret_cast<__nv_bfloat16*>(p.out) + (int64_t)m * p.ldo + n, v);
        }
      } else {  // EPI_HEAD: h = ReLU(acc + b) kept in fp32, dotted with the head weights
#pragma unroll
        for (int j = 0; j < 16; ++j) z = fmaf(fmaxf(v[j] + __ldg(p.bias + n + j), 0.f), __ldg(p.head_w + n + j), z);
      }
    }
    if constexpr (EPI == EPI_HEAD) {
      if (live) p.scores[m] = sigmoid_f32(z + p.head_b);
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) ptx::tmem_dealloc(tmem, C::TMEM_COLS);
}

template <int BN, int EPI>
cudaError_t launch_t(const CUtensorMap* tmA, const CUtensorMap* tmB, int M, int N, int K, const EpiParams& p,
                     cudaStream_t s) {
  using C = Cfg<BN>;
  auto kern = gemm_bf16_kernel<BN, EPI>;
  static bool attr_done = false;
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return e;
    attr_done = true;
  }
  dim3 grid(N / BN, (M + BM - 1) / BM);
  kern<<<grid, kThreads, C::SMEM, s>>>(*tmA, *tmB, p, M, K);
  return cudaGetLastError();
}

template <int BN>
cudaError_t launch_bn(const CUtensorMap* tmA, const CUtensorMap* tmB, int M, int N, int K, Epi epi,
                      const EpiParams& p, cudaStream_t s) {
  switch (epi) {
    case EPI_STORE: return launch_t<BN, EPI_STORE>(tmA, tmB, M, N, K, p, s);
    case EPI_BIAS_RELU: return launch_t<BN, EPI_BIAS_RELU>(tmA, tmB, M, N, K, p, s);
    case EPI_CROSS: return launch_t<BN, EPI_CROSS>(tmA, tmB, M, N, K, p, s);
    case EPI_HEAD: return launch_t<BN, EPI_HEAD>(tmA, tmB, M, N, K, p, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace

cudaError_t launch_gemm_bf16(const CUtensorMap* tmA, const CUtensorMap* tmB, int M, int N, int K, int BN, Epi epi,
                             const EpiParams& p, cudaStream_t s) {
  if (M <= 0) return cudaSuccess;
  if (K % BK || N % BN || (epi == EPI_HEAD && BN != N)) return cudaErrorInvalidValue;
  switch (BN) {
    case 64: return launch_bn<64>(tmA, tmB, M, N, K, epi, p, s);
    case 128: return launch_bn<128>(tmA, tmB, M, N, K, epi, p, s);
    case 256: return launch_bn<256>(tmA, tmB, M, N, K, epi, p, s);
  }
  return cudaErrorInvalidValue;
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
