// Random-row gather ceiling on this GPU: N lookups of uniformly random rows (row_bytes each) out of a table of
// `table_mb` MB, each row read by row_bytes/16 lanes with one 16-byte non-coherent load (no L1 allocation), the
// values summed per lane group and one 16-byte result stored per lookup (so the loads are not dead).  This is
// the memory-system ceiling the embedding gather (embed_bag_kernel, same access pattern on uniform indices) is
// measured against.  Usage: rand_rows [row_bytes=128] [n_lookups=561152] [table_mb=1536] [unroll=1]
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <random>
#include <cuda_runtime.h>

template <int U>
__global__ void __launch_bounds__(256) gather(const uint8_t* __restrict__ tab, const int32_t* __restrict__ idx,
                                              int64_t n, int row_bytes, uint4* __restrict__ out) {
  const int lpr = row_bytes / 16;
  const int sub = threadIdx.x % lpr;
  const int64_t groups = (int64_t)gridDim.x * blockDim.x / lpr;
  for (int64_t g = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / lpr; g * U < n; g += groups) {
    uint4 acc = make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t j = g * U + u;
      if (j < n) {
        const int64_t r = __ldg(idx + j);
        uint4 v;
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                     : "l"(tab + r * row_bytes + sub * 16));
        acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
      }
    }
    out[g * lpr + sub] = acc;
  }
}

int main(int argc, char** argv) {
  const int row_bytes = argc > 1 ? atoi(argv[1]) : 128;
  const int64_t n = argc > 2 ? atoll(argv[2]) : 561152;
  const int64_t table_mb = argc > 3 ? atoll(argv[3]) : 1536;
  const int U = argc > 4 ? atoi(argv[4]) : 1;
  const int64_t rows = table_mb * (1 << 20) / row_bytes;
  uint8_t* tab;
  int32_t* didx;
  uint4* out;
  cudaMalloc(&tab, rows * row_bytes);
  cudaMemset(tab, 1, rows * row_bytes);
  std::vector<int32_t> h(n);
  std::mt19937_64 rng(7);
  for (auto& x : h) x = (int32_t)(rng() % rows);
  cudaMalloc(&didx, n * 4);
  cudaMemcpy(didx, h.data(), n * 4, cudaMemcpyHostToDevice);
  const int lpr = row_bytes / 16;
  cudaMalloc(&out, ((n + U - 1) / U) * lpr * 16 + 4096);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int64_t groups_needed = (n + U - 1) / U;
  const int64_t blocks_full = (groups_needed * lpr + 255) / 256;
  for (int cap : {0, 8, 16, 32}) {  // 0 = one lookup group per lane group (no grid-stride), else CTAs per SM
    const int64_t blocks = cap ? std::min<int64_t>(blocks_full, (int64_t)sms * cap) : blocks_full;
    auto launch = [&]() {
      if (U == 1) gather<1><<<(unsigned)blocks, 256>>>(tab, didx, n, row_bytes, out);
      else if (U == 2) gather<2><<<(unsigned)blocks, 256>>>(tab, didx, n, row_bytes, out);
      else gather<4><<<(unsigned)blocks, 256>>>(tab, didx, n, row_bytes, out);
    };
    for (int i = 0; i < 3; ++i) launch();
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int reps = 50;
    cudaEventRecord(a);
    for (int i = 0; i < reps; ++i) launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const double us = ms * 1e3 / reps;
    const double bytes = (double)n * (row_bytes + 4) + (double)groups_needed * lpr * 16;
    printf("{\"row_bytes\": %d, \"lookups\": %lld, \"table_mb\": %lld, \"unroll\": %d, \"ctas_per_sm_cap\": %d, "
           "\"us\": %.2f, \"GBps\": %.1f, \"rows_per_us\": %.0f}\n",
           row_bytes, (long long)n, (long long)table_mb, U, cap, us, bytes / us / 1e3, n / us);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    printf("error %s\n", cudaGetErrorString(e));
    return 1;
  }
  return 0;
}
