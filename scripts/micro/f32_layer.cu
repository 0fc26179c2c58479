// Why does config 1's 141 x 141 fp32 layer take ~3.6 us inside dense_f32_kernel?  Time one layer's loop (R = 2 rows,
// 256 threads, weights W^T and activations already in shared memory) in clock cycles, for a few loop shapes.
// Usage: f32_layer
#include <cstdio>
#include <cuda_runtime.h>

constexpr int R = 2, N = 141, LD = 144;

template <int VAR>
__global__ void __launch_bounds__(256) layer_kernel(const float* __restrict__ gw, float* out, long long* cyc, int reps) {
  extern __shared__ float smf[];
  float* ws = smf;
  float* in = smf + N * N;
  float* o = in + R * LD;
  for (int i = threadIdx.x; i < N * N; i += blockDim.x) ws[i] = gw[i];
  for (int i = threadIdx.x; i < R * LD; i += blockDim.x) in[i] = 0.001f * i;
  __syncthreads();
  long long t0 = clock64();
  for (int rep = 0; rep < reps; ++rep) {
    if (VAR == 0) {  // the kernel's loop: one output per thread, k serial, unroll 4
      for (int j = threadIdx.x; j < N; j += blockDim.x) {
        float acc[R] = {0.f, 0.f};
#pragma unroll 4
        for (int k = 0; k < N; ++k) {
          const float w = ws[k * N + j];
#pragma unroll
          for (int r = 0; r < R; ++r) acc[r] = fmaf(in[r * LD + k], w, acc[r]);
        }
        for (int r = 0; r < R; ++r) o[r * LD + j] = acc[r];
      }
    } else if (VAR == 1) {  // same, 4 independent partial sums per row (breaks the 141-long FMA chain)
      for (int j = threadIdx.x; j < N; j += blockDim.x) {
        float acc[R][4] = {};
        int k = 0;
        for (; k + 4 <= N; k += 4) {
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const float w = ws[(k + u) * N + j];
#pragma unroll
            for (int r = 0; r < R; ++r) acc[r][u] = fmaf(in[r * LD + k + u], w, acc[r][u]);
          }
        }
        for (; k < N; ++k)
          for (int r = 0; r < R; ++r) acc[r][0] = fmaf(in[r * LD + k], ws[k * N + j], acc[r][0]);
        for (int r = 0; r < R; ++r) o[r * LD + j] = (acc[r][0] + acc[r][1]) + (acc[r][2] + acc[r][3]);
      }
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = (t1 - t0) / reps;
  if (threadIdx.x < R * LD) out[blockIdx.x * R * LD + threadIdx.x] = o[threadIdx.x];
}

int main() {
  float* gw;
  float* out;
  long long* cyc;
  cudaMalloc(&gw, N * N * 4);
  cudaMemset(gw, 0, N * N * 4);
  cudaMalloc(&out, 128 * R * LD * 4);
  cudaMalloc(&cyc, 128 * 8);
  long long h[128];
  const int smem = (N * N + 2 * R * LD) * 4;
  cudaFuncSetAttribute(layer_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(layer_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  layer_kernel<0><<<128, 256, smem>>>(gw, out, cyc, 100);
  cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost);
  printf("{\"variant\": \"serial k, 1 output/thread\", \"cycles_per_layer\": %lld, \"us\": %.2f}\n", h[0], h[0] / 1965.0);
  layer_kernel<1><<<128, 256, smem>>>(gw, out, cyc, 100);
  cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost);
  printf("{\"variant\": \"4 partial sums per row\", \"cycles_per_layer\": %lld, \"us\": %.2f}\n", h[0], h[0] / 1965.0);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
