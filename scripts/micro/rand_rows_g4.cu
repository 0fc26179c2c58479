// Random-row gather through TMA tile::gather4 (sm_100a): the same workload as rand_rows.cu -- N lookups of
// uniformly random 128-byte rows of a 1.5 GB table -- with the rows landing in a shared-memory ring by
// cp.async.bulk.tensor.2d.tile::gather4 (4 rows per instruction) instead of per-lane 16-byte loads, so rows in
// flight cost ring bytes, not registers.  Warp 0 reads the row ids (one coalesced load per 32) and one lane issues
// the gathers; warps 1-3 fold each landed stage (xor, 16 bytes per lane) and free it.
// Usage: rand_rows_g4 [n_lookups=8000000] [table_mb=1536] [stages=8] [ctas_per_sm=4]
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

constexpr int ROWB = 128;            // bytes per row (64 bf16)
constexpr int ROWS_PER_STAGE = 32;   // 8 gather4 per stage
constexpr int STAGE_BYTES = ROWS_PER_STAGE * ROWB;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(128) g4_kernel(const __grid_constant__ CUtensorMap tm, const int32_t* __restrict__ idx,
                                                 int64_t n, int stages, uint4* __restrict__ out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + stages * STAGE_BYTES);
  uint64_t* empty = full + stages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&full[s])), "r"(1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&empty[s])), "r"(3));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t chunks = (n + ROWS_PER_STAGE - 1) / ROWS_PER_STAGE;
  if (warp == 0) {
    int k = 0;
    // row ids of the next PF chunks are loaded ahead (the id load -> gather chain otherwise serialises each stage)
    constexpr int PF = 4;
    int ids[PF];
#pragma unroll
    for (int p = 0; p < PF; ++p) {
      const int64_t j = (blockIdx.x + (int64_t)p * gridDim.x) * ROWS_PER_STAGE + lane;
      ids[p] = j < n ? __ldg(idx + j) : 0;
    }
    for (int64_t c = blockIdx.x; c < chunks; c += gridDim.x, ++k) {
      const int s = k % stages;
      const int my = ids[0];
#pragma unroll
      for (int p = 0; p + 1 < PF; ++p) ids[p] = ids[p + 1];
      {
        const int64_t j = (c + (int64_t)PF * gridDim.x) * ROWS_PER_STAGE + lane;
        ids[PF - 1] = j < n ? __ldg(idx + j) : 0;
      }
      if (k >= stages) {
        const uint32_t par = ((k / stages) - 1) & 1;
        asm volatile("{\n.reg .pred p;\nW1:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W1;\n}" ::"r"(
                         smem_u32(&empty[s])),
                     "r"(par)
                     : "memory");
      }
      int r[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) r[i] = __shfl_sync(0xffffffffu, my, i);
      if (lane == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[s])), "r"(STAGE_BYTES)
                     : "memory");
        uint8_t* dst = sm + s * STAGE_BYTES;
#pragma unroll
        for (int g = 0; g < 8; ++g)
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
              "%4, %5, %6, %7}], [%2];" ::"r"(smem_u32(dst + g * 4 * ROWB)),
              "l"(&tm), "r"(smem_u32(&full[s])), "r"(0), "r"(r[4 * g]), "r"(r[4 * g + 1]), "r"(r[4 * g + 2]),
              "r"(r[4 * g + 3])
              : "memory");
      }
      __syncwarp();
    }
  } else {
    uint4 acc = make_uint4(0, 0, 0, 0);
    int k = 0;
    const int t = threadIdx.x - 32;  // 96 consumer threads: 256 16-byte chunks per stage
    for (int64_t c = blockIdx.x; c < chunks; c += gridDim.x, ++k) {
      const int s = k % stages;
      asm volatile("{\n.reg .pred p;\nW2:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W2;\n}" ::"r"(
                       smem_u32(&full[s])),
                   "r"((uint32_t)((k / stages) & 1))
                   : "memory");
      const uint4* st = reinterpret_cast<const uint4*>(sm + s * STAGE_BYTES);
      for (int i = t; i < STAGE_BYTES / 16; i += 96) {
        const uint4 v = st[i];
        acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
      }
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[s])) : "memory");
    }
    out[blockIdx.x * 96 + t] = acc;
  }
}

int main(int argc, char** argv) {
  const int64_t n = argc > 1 ? atoll(argv[1]) : 8000000;
  const int64_t table_mb = argc > 2 ? atoll(argv[2]) : 1536;
  const int stages = argc > 3 ? atoi(argv[3]) : 8;
  const int cps = argc > 4 ? atoi(argv[4]) : 4;
  const int64_t rows = table_mb * (1 << 20) / ROWB;
  uint8_t* tab;
  cudaMalloc(&tab, rows * ROWB);
  cudaMemset(tab, 1, rows * ROWB);
  std::vector<int32_t> h(n);
  std::mt19937_64 rng(7);
  for (auto& x : h) x = (int32_t)(rng() % rows);
  int32_t* didx;
  cudaMalloc(&didx, n * 4);
  cudaMemcpy(didx, h.data(), n * 4, cudaMemcpyHostToDevice);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint4* out;
  cudaMalloc(&out, (size_t)sms * cps * 96 * 16);
  // tensor map: [rows][64] bf16, box {64, 1} (gather4 loads 4 such rows)
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto encode = reinterpret_cast<CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                                              CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                              CUtensorMapFloatOOBfill)>(fn);
  CUtensorMap tm;
  cuuint64_t gdim[2] = {64, (cuuint64_t)rows};
  cuuint64_t gstr[1] = {ROWB};
  cuuint32_t box[2] = {64, 1};
  cuuint32_t es[2] = {1, 1};
  CUresult cr = encode(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, tab, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                       CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) {
    printf("encode failed %d\n", (int)cr);
    return 1;
  }
  const size_t smem = (size_t)stages * STAGE_BYTES + 2 * stages * 8;
  cudaFuncSetAttribute(g4_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int blocks = sms * cps;
  for (int i = 0; i < 3; ++i) g4_kernel<<<blocks, 128, smem>>>(tm, didx, n, stages, out);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int reps = 20;
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) g4_kernel<<<blocks, 128, smem>>>(tm, didx, n, stages, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  cudaError_t e = cudaGetLastError();
  const double us = ms * 1e3 / reps;
  printf("{\"gather4\": true, \"lookups\": %lld, \"stages\": %d, \"ctas_per_sm\": %d, \"smem_per_cta\": %zu, \"us\": %.2f, "
         "\"GBps\": %.1f, \"rows_per_us\": %.0f, \"err\": \"%s\"}\n",
         (long long)n, stages, cps, smem, us, (double)n * (ROWB + 4) / us / 1e3, n / us, cudaGetErrorString(e));
  return e == cudaSuccess ? 0 : 1;
}
