// TMA ingest microbenchmark: every CTA (one per SM) streams 16 KB tiles (box 64 x 128 bf16, 128B swizzle)
// through an S-stage mbarrier ring with no compute.  share = k: groups of k consecutive CTAs read the
// same tile sequence at the same time (as the N-tiles of one GEMM row block do).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
#include "../../paper_2605_29232_b200/csrc/cvr_ptx.cuh"
using namespace cvr;
template <int S>
__global__ void __launch_bounds__(64, 1) tma_stream(const __grid_constant__ CUtensorMap tm, int tiles, int share,
                                                     int rows_tiles, unsigned long long* sink) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + S * 16384);
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) ptx::mbar_init(&full[s], 1);
    ptx::fence_barrier_init();
  }
  __syncthreads();
  const int grp = blockIdx.x / share;
  if (threadIdx.x == 0) {
    for (int i = 0; i < tiles + S; ++i) {
      if (i >= S) ptx::mbar_wait(&full[(i - S) % S], ((i - S) / S) & 1);
      if (i < tiles) {
        const int s = i % S;
        const int t = (grp * 7919 + i) % (rows_tiles * 27);
        ptx::mbar_arrive_expect_tx(&full[s], 16384);
        ptx::tma_load_2d(sm + s * 16384, &tm, &full[s], (t % 27) * 64, (t / 27) * 128);
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0 && sink) sink[blockIdx.x] = 1;
}
int main() {
  const int rows = 32768, cols = 1728;  // 113 MB bf16 (> L2) or use fewer rows for L2-resident
  for (int rr : {4096, 32768}) {
    void* buf;
    cudaMalloc(&buf, (size_t)rr * cols * 2);
    cudaMemset(buf, 1, (size_t)rr * cols * 2);
    void* fn;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
    CUtensorMap tm;
    cuuint64_t gd[2] = {(cuuint64_t)cols, (cuuint64_t)rr}, gs[1] = {(cuuint64_t)cols * 2};
    cuuint32_t box[2] = {64, 128}, es[2] = {1, 1};
    enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, gd, gs, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int smem = 13 * 16384 + 2048;
    cudaFuncSetAttribute(tma_stream<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(tma_stream<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(tma_stream<13>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int w = 0; w < 50; ++w) tma_stream<8><<<148, 64, smem>>>(tm, 2000, 1, rr / 128, nullptr);  // warm clocks
    cudaDeviceSynchronize();
    for (int grid : {148}) {
      for (int share : {1, 4, 16, 37, 148}) {
        const int tiles = 2000, st = 8;
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        for (int w = 0; w < 5; ++w) {
          cudaEventRecord(a);
          tma_stream<8><<<grid, 64, smem>>>(tm, tiles, share, rr / 128, nullptr);
          cudaEventRecord(b);
          cudaEventSynchronize(b);
        }
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const double bytes = (double)grid * tiles * 16384;
        printf("rows %5d grid %3d stages %d share %3d: %.2f TB/s (%.1f GB/s per SM)\n", rr, grid, st, share,
               bytes / ms / 1e9, bytes / ms / 1e6 / grid);
      }
    }
    cudaFree(buf);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
