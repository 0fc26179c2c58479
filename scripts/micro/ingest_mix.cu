// Per-SM ingest: TMA alone, LDG alone, and TMA + LDG together (L2-resident source), one CTA per SM.
// Answers whether the ~47 B/clk/SM TMA ceiling is the SM's port limit or the TMA engine's.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include "../../paper_2605_29232_b200/csrc/cvr_ptx.cuh"
using namespace cvr;
constexpr int S = 5;
__global__ void __launch_bounds__(512, 1) mix(const __grid_constant__ CUtensorMap tm, const uint4* src, size_t n16,
                                              int tma_tiles, int ldg_iters, int ldg_warps, unsigned long long* sink,
                                              int mode) {  // mode 0: LDG warps, 1: cp.async warps, 2: 2nd TMA warp
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + 2 * S * 16384);
  if (threadIdx.x == 0) {
    for (int s = 0; s < 2 * S; ++s) ptx::mbar_init(&full[s], 1);
    ptx::fence_barrier_init();
  }
  __syncthreads();
  unsigned long long c0 = clock64(), g0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    if (lane == 0) {
      for (int i = 0; i < tma_tiles + S; ++i) {
        if (i >= S) ptx::mbar_wait(&full[(i - S) % S], ((i - S) / S) & 1);
        if (i < tma_tiles) {
          const int s = i % S;
          const int t = (blockIdx.x * 7919 + i) % (32 * 27);
          ptx::mbar_arrive_expect_tx(&full[s], 16384);
          ptx::tma_load_2d(sm + s * 16384, &tm, &full[s], (t % 27) * 64, (t / 27) * 128);
        }
      }
    }
  } else if (mode == 2 && warp == 1) {
    if (lane == 0) {
      uint64_t* f2 = full + S;
      uint8_t* sm2 = sm + S * 16384;
      for (int i = 0; i < tma_tiles + S; ++i) {
        if (i >= S) ptx::mbar_wait(&f2[(i - S) % S], ((i - S) / S) & 1);
        if (i < tma_tiles) {
          const int s = i % S;
          const int t = (blockIdx.x * 7919 + 5 * i + 3) % (32 * 27);
          ptx::mbar_arrive_expect_tx(&f2[s], 16384);
          ptx::tma_load_2d(sm2 + s * 16384, &tm, &f2[s], (t % 27) * 64, (t / 27) * 128);
        }
      }
    }
  } else if (mode == 1 && warp <= ldg_warps) {
    // cp.async 16 B per lane into a private 8 KB smem window per warp, 8 in flight per lane, then wait
    uint8_t* win = sm + S * 16384 + (warp - 1) * 4096;
    size_t base = ((size_t)blockIdx.x * 977 * 512 + (warp - 1) * 32 * 8) % (n16 - 4096);
    for (int it = 0; it < ldg_iters; ++it) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const uint32_t d = ptx::smem_u32(win + ((u * 32 + lane) & 255) * 16);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src + base + u * 32 + lane) : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
      asm volatile("cp.async.wait_group 2;" ::: "memory");
      base += (size_t)ldg_warps * 256;
      if (base + 256 > n16) base = lane & 7;
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
  } else if (mode == 0 && warp <= ldg_warps) {
    uint4 acc = make_uint4(0, 0, 0, 0);
    size_t base = ((size_t)blockIdx.x * 977 * 512 + (warp - 1) * 32 * 8) % (n16 - 4096);
    for (int it = 0; it < ldg_iters; ++it) {
      uint4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = ptx::ld_nc_v4(src + base + u * 32 + lane);
#pragma unroll
      for (int u = 0; u < 8; ++u) { acc.x ^= v[u].x; acc.y ^= v[u].y; acc.z += v[u].z; acc.w += v[u].w; }
      base += (size_t)ldg_warps * 256;
      if (base + 256 > n16) base = lane & 7;
    }
    if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x12345678u) sink[blockIdx.x] = 1;
  }
  __syncthreads();
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    unsigned long long c1 = clock64(), g1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
    sink[1000] = c1 - c0;
    sink[1001] = g1 - g0;
  }
}
int main() {
  const int rr = 4096, cols = 1728;
  void* buf;
  cudaMalloc(&buf, (size_t)rr * cols * 2);
  cudaMemset(buf, 1, (size_t)rr * cols * 2);
  unsigned long long* sink;
  cudaMalloc(&sink, 8 * 1024);
  void* fn;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  CUtensorMap tm;
  cuuint64_t gd[2] = {(cuuint64_t)cols, (cuuint64_t)rr}, gs[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box[2] = {64, 128}, es[2] = {1, 1};
  enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, gd, gs, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const int smem = 2 * S * 16384 + 2048;
  cudaFuncSetAttribute(mix, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const size_t n16 = (size_t)rr * cols * 2 / 16;
  struct Case { int tma, ldg, warps, mode; const char* name; } cases[] = {
      {6000, 0, 0, 0, "TMA only"}, {6000, 0, 0, 2, "2 TMA warps"}, {0, 2000, 8, 0, "LDG only (8 warps)"},
      {6000, 2000, 8, 0, "TMA + LDG (8 warps)"}, {0, 2000, 8, 1, "cp.async (8 warps)"},
      {6000, 2000, 8, 1, "TMA + cp.async (8w)"}, {6000, 2000, 4, 1, "TMA + cp.async (4w)"}};
  {  // warm the clocks: ~300 ms of TMA streaming
    for (int w = 0; w < 100; ++w) mix<<<148, 512, smem>>>(tm, (const uint4*)buf, n16, 6000, 0, 0, sink, 0);
    cudaDeviceSynchronize();
  }
  for (int grid : {16, 148}) {
    for (auto& c : cases) {
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      float ms = 0;
      for (int w = 0; w < 30; ++w) {
        cudaEventRecord(a);
        mix<<<grid, 512, smem>>>(tm, (const uint4*)buf, n16, c.tma, c.ldg, c.warps, sink, c.mode);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
      }
      const double bytes = (double)grid * ((double)c.tma * 16384 * (c.mode == 2 ? 2 : 1) +
                                           (double)c.ldg * c.warps * 32 * 8 * 16);
      unsigned long long h[2];
      cudaMemcpy(h, sink + 1000, 16, cudaMemcpyDeviceToHost);
      printf("grid %3d %-22s: %.3f ms, %.1f GB/s per SM, SM clock %.0f MHz, %.1f B/clk/SM\n", grid, c.name, ms,
             bytes / ms / 1e6 / grid, (double)h[0] / (double)h[1] * 1e3,
             bytes / grid / ((double)h[0] / (double)h[1] * 1e9 * ms / 1e3));
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
