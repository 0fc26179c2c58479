// dense_f32.cu -- K3: the fp32 dense stage of config 1 in one fused SIMT kernel.
//
//   S5 full-rank cross  x_{l+1} = x0 * (W_l x_l + b_l) + x_l      PAPER.md:116-119 (eq:dcnv2)
//   S6 MLP              h_{i+1} = ReLU(M_i h_i + c_i)
//   S7 head             score  = sigmoid(m . h + c)               BASELINE.json north star
//
// True fp32 FFMA (no TF32: SURVEY.md A17, the 1e-5 gate).  One CTA owns R rows, keeps x0, x_l
// and the next activation in shared memory, and reads the weights as W^T ([in][out], repacked
// by cvr_load_weights) so the 256 threads of a CTA read one contiguous weight row per k.
// Per-row work is independent of the batch (batch invariance).
#include <algorithm>

#include "cvr_kernels.cuh"

namespace cvr {
namespace {

constexpr int R = 4;  // rows per CTA (B = 256 -> 64 CTAs)

__device__ __forceinline__ float sigmoid_f32(float z) {
  if (z >= 0.f) return 1.f / (1.f + expf(-z));
  const float e = expf(z);
  return e / (1.f + e);
}

// out[r][j] = act(sum_k in[r][k] * WT[k][j] + bias[j]) (+ cross epilogue).  The layer's W^T is first
// staged in shared memory with coalesced loads (one L2 round trip for the whole matrix instead of one
// dependent load per k), then every thread runs its k loop on shared memory.
template <bool CROSS>
__device__ void layer(const float* __restrict__ in, int n_in, float* __restrict__ out, int n_out, int ld,
                      const float* __restrict__ WT, const float* __restrict__ bias, const float* __restrict__ x0s,
                      float* __restrict__ ws) {
  const int n = n_in * n_out;
  const int n4 = n >> 2;  // float4 body (WT is 256-byte aligned in the workspace), scalar tail
  const float4* src4 = reinterpret_cast<const float4*>(WT);
  float4* dst4 = reinterpret_cast<float4*>(ws);
#pragma unroll 8
  for (int i = threadIdx.x; i < n4; i += blockDim.x) dst4[i] = __ldg(src4 + i);
  for (int i = 4 * n4 + threadIdx.x; i < n; i += blockDim.x) ws[i] = __ldg(WT + i);
  __syncthreads();
  for (int j = threadIdx.x; j < n_out; j += blockDim.x) {
    float acc[R];
#pragma unroll
    for (int r = 0; r < R; ++r) acc[r] = 0.f;
#pragma unroll 4
    for (int k = 0; k < n_in; ++k) {
      const float w = ws[k * n_out + j];
#pragma unroll
      for (int r = 0; r < R; ++r) acc[r] = fmaf(in[r * ld + k], w, acc[r]);
    }
    const float bj = __ldg(bias + j);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (CROSS)
        out[r * ld + j] = x0s[r * ld + j] * (acc[r] + bj) + in[r * ld + j];
      else
        out[r * ld + j] = fmaxf(acc[r] + bj, 0.f);
    }
  }
}

__global__ void __launch_bounds__(256) dense_f32_kernel(const DenseF32Args a, int ld) {
  extern __shared__ float sm[];
  float* x0s = sm;
  float* bufA = sm + R * ld;
  float* bufB = sm + 2 * R * ld;
  float* ws = sm + 3 * R * ld;  // staged weights of the current layer
  const int row0 = blockIdx.x * R;
  for (int i = threadIdx.x; i < R * a.W; i += blockDim.x) {
    const int r = i / a.W, c = i - r * a.W;
    const float v = (row0 + r < a.B) ? a.x0[(int64_t)(row0 + r) * a.x0_ld + c] : 0.f;
    x0s[r * ld + c] = v;
    bufA[r * ld + c] = v;
  }
  __syncthreads();
  float* cur = bufA;
  float* nxt = bufB;
  for (int l = 0; l < a.n_cross; ++l) {
    layer<true>(cur, a.W, nxt, a.W, ld, a.WT[l], a.bias[l], x0s, ws);
    __syncthreads();
    float* t = cur; cur = nxt; nxt = t;
  }
  for (int i = 0; i < a.n_mlp; ++i) {
    layer<false>(cur, a.dims[i], nxt, a.dims[i + 1], ld, a.MT[i], a.mb[i], nullptr, ws);
    __syncthreads();
    float* t = cur; cur = nxt; nxt = t;
  }
  const int hn = a.dims[a.n_mlp];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int r = warp; r < R; r += blockDim.x >> 5) {
    float s = 0.f;
    for (int k = lane; k < hn; k += 32) s = fmaf(cur[r * ld + k], __ldg(a.head_w + k), s);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0 && row0 + r < a.B) a.scores[row0 + r] = sigmoid_f32(s + __ldg(a.head_b));
  }
}

}  // namespace

cudaError_t launch_dense_f32(const DenseF32Args& a, cudaStream_t s) {
  if (a.B <= 0) return cudaSuccess;
  int ld = a.W;
  size_t wmax = (size_t)a.W * a.W * (a.n_cross > 0);
  for (int i = 0; i <= a.n_mlp; ++i) ld = a.dims[i] > ld ? a.dims[i] : ld;
  for (int i = 0; i < a.n_mlp; ++i) wmax = std::max(wmax, (size_t)a.dims[i] * a.dims[i + 1]);
  ld = (ld + 3) & ~3;
  const size_t smem = ((size_t)3 * R * ld + wmax) * sizeof(float);
  if (smem > 220 * 1024) return cudaErrorInvalidValue;
  static size_t attr_set = 0;
  if (smem > 48 * 1024 && smem > attr_set) {
    cudaError_t e = cudaFuncSetAttribute(dense_f32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr_set = smem;
  }
  dense_f32_kernel<<<(a.B + R - 1) / R, 256, smem, s>>>(a, ld);
  return cudaGetLastError();
}

}  // namespace cvr
