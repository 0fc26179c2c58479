// dense_f32.cu -- K3: the fp32 dense stage of config 1 in one fused SIMT kernel.
//
//   S5 full-rank cross  x_{l+1} = x0 * (W_l x_l + b_l) + x_l      PAPER.md:116-119 (eq:dcnv2)
//   S6 MLP              h_{i+1} = ReLU(M_i h_i + c_i)
//   S7 head             score  = sigmoid(m . h + c)               BASELINE.json north star
//
// True fp32 FFMA (no TF32: SURVEY.md A17, the 1e-5 gate).  One CTA owns R rows, keeps x0, x_l
// and the next activation in shared memory, and reads the weights as W^T ([in][out], repacked
// by cvr_load_weights) so the 256 threads of a CTA read one contiguous weight row per k.  When every layer's
// W^T fits in shared memory (config 1) all of them are bulk-copied at kernel start (dense_f32_resident_kernel);
// otherwise each layer's W^T is staged by cp.async one layer ahead (double buffer, dense_f32_kernel).
// Per-row work is independent of the batch (batch invariance).
#include <algorithm>

#include "cvr_kernels.cuh"
#include "cvr_ptx.cuh"

namespace cvr {
namespace {

constexpr int R = 2;  // rows per CTA (B = 256 -> 128 CTAs)

__device__ __forceinline__ float sigmoid_f32(float z) {
  if (z >= 0.f) return 1.f / (1.f + expf(-z));
  const float e = expf(z);
  return e / (1.f + e);
}

__device__ __forceinline__ void cp_async16(float* dst, const float* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async4(float* dst, const float* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// stage a layer's W^T [n_in][n_out] (workspace: 256-byte aligned) into shared memory with cp.async (one group)
__device__ void stage(float* __restrict__ ws, const float* __restrict__ WT, int n) {
  const int n4 = n >> 2;
  for (int i = threadIdx.x; i < n4; i += blockDim.x) cp_async16(ws + 4 * i, WT + 4 * i);
  for (int i = 4 * n4 + threadIdx.x; i < n; i += blockDim.x) cp_async4(ws + i, WT + i);
  cp_commit();
}

// out[r][j] = act(sum_k in[r][k] * WT[k][j] + bias[j]) (+ cross epilogue) from the staged W^T in ws: one output
// column per thread (consecutive threads read consecutive weight words), 4 independent partial sums per row (k mod
// 4) added as (s0 + s1) + (s2 + s3), so the 141-long dependent FMA chain becomes four ~35-long ones
// (scripts/micro/f32_layer.cu: 1.40 -> 1.06 us per 141 x 141 layer; c1's dense stage 15.4 -> 14.4 us).
template <bool CROSS>
__device__ void layer4(const float* __restrict__ in, int n_in, float* __restrict__ out, int n_out, int ld,
                       const float* __restrict__ ws, const float* __restrict__ bias, const float* __restrict__ x0s) {
  for (int j = threadIdx.x; j < n_out; j += blockDim.x) {
    float acc[R][4];
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int u = 0; u < 4; ++u) acc[r][u] = 0.f;
    int k = 0;
    for (; k + 4 <= n_in; k += 4) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float w = ws[(k + u) * n_out + j];
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r][u] = fmaf(in[r * ld + k + u], w, acc[r][u]);
      }
    }
    for (; k < n_in; ++k) {
      const float w = ws[k * n_out + j];
#pragma unroll
      for (int r = 0; r < R; ++r) acc[r][k & 3] = fmaf(in[r * ld + k], w, acc[r][k & 3]);
    }
    const float bj = __ldg(bias + j);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const float sum = (acc[r][0] + acc[r][1]) + (acc[r][2] + acc[r][3]);
      if (CROSS)
        out[r * ld + j] = x0s[r * ld + j] * (sum + bj) + in[r * ld + j];
      else
        out[r * ld + j] = fmaxf(sum + bj, 0.f);
    }
  }
}

// Weights of layer i + 1 stream into the second shared-memory buffer (cp.async) while layer i computes,
// so a layer costs max(staging, math) rather than their sum.
__global__ void __launch_bounds__(256) dense_f32_kernel(const DenseF32Args a, int ld, int wmax) {
  extern __shared__ float sm[];
  // executor graphs: this batch's rows / scores pointer from the per-call block (grid sized for max_batch)
  const int B = a.call ? a.call->B : a.B;
  float* const scores = a.call ? a.call->scores : a.scores;
  if ((int)blockIdx.x * R >= B) return;
  float* x0s = sm;
  float* bufA = sm + R * ld;
  float* bufB = sm + 2 * R * ld;
  float* wbuf[2] = {sm + 3 * R * ld, sm + 3 * R * ld + wmax};
  const int n_layers = a.n_cross + a.n_mlp;
  auto wt = [&](int i) { return i < a.n_cross ? a.WT[i] : a.MT[i - a.n_cross]; };
  auto wn = [&](int i) {
    return i < a.n_cross ? a.W * a.W : a.dims[i - a.n_cross] * a.dims[i - a.n_cross + 1];
  };
  if (n_layers > 0) stage(wbuf[0], wt(0), wn(0));
  const int row0 = blockIdx.x * R;
  for (int i = threadIdx.x; i < R * a.W; i += blockDim.x) {
    const int r = i / a.W, c = i - r * a.W;
    const float v = (row0 + r < B) ? a.x0[(int64_t)(row0 + r) * a.x0_ld + c] : 0.f;
    x0s[r * ld + c] = v;
    bufA[r * ld + c] = v;
  }
  float* cur = bufA;
  float* nxt = bufB;
  for (int l = 0; l < n_layers; ++l) {
    if (l + 1 < n_layers) {
      stage(wbuf[(l + 1) & 1], wt(l + 1), wn(l + 1));
      cp_wait<1>();  // this thread's copies of layer l have landed
    } else {
      cp_wait<0>();
    }
    __syncthreads();  // everyone's copies of layer l (and the activations) are visible
    if (l < a.n_cross) {
      layer4<true>(cur, a.W, nxt, a.W, ld, wbuf[l & 1], a.bias[l], x0s);
    } else {
      const int i = l - a.n_cross;
      layer4<false>(cur, a.dims[i], nxt, a.dims[i + 1], ld, wbuf[l & 1], a.mb[i], nullptr);
    }
    __syncthreads();  // layer l's weights and activations consumed before they are overwritten
    float* t = cur; cur = nxt; nxt = t;
  }
  const int hn = a.dims[a.n_mlp];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int r = warp; r < R; r += blockDim.x >> 5) {
    float s = 0.f;
    for (int k = lane; k < hn; k += 32) s = fmaf(cur[r * ld + k], __ldg(a.head_w + k), s);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0 && row0 + r < B) scores[row0 + r] = sigmoid_f32(s + __ldg(a.head_b));
  }
}

// Every layer's W^T resident at once (config 1: 203 KB of the 227 KB): all weight copies are issued at kernel start
// (one bulk copy per layer, one mbarrier each), so layer l waits only for its own weights and the later layers'
// copies stream in while it computes.  Measured on c1 (B = 256): dense stage 20.6 -> 15.4 us.  (The double-buffered
// staging, one layer ahead, paid ~4.5 us per 141 x 141 layer against ~1.4 us of math; multicasting each layer
// across clusters of 2 / 4 CTAs -- the L2 then serves each byte once per cluster -- measured 21.3 / 20.8 us.)
__global__ void __launch_bounds__(256) dense_f32_resident_kernel(const DenseF32Args a, int ld) {
  extern __shared__ __align__(16) float sm[];
  __shared__ uint64_t wbar[kMaxLayers];
  // executor graphs: this batch's rows / scores pointer from the per-call block (grid sized for max_batch)
  const int B = a.call ? a.call->B : a.B;
  float* const scores = a.call ? a.call->scores : a.scores;
  if ((int)blockIdx.x * R >= B) return;
  float* x0s = sm;
  float* bufA = sm + R * ld;
  float* bufB = sm + 2 * R * ld;
  float* wbase = sm + 3 * R * ld;
  const int n_layers = a.n_cross + a.n_mlp;
  auto wt = [&](int i) { return i < a.n_cross ? a.WT[i] : a.MT[i - a.n_cross]; };
  auto wn = [&](int i) {
    return i < a.n_cross ? a.W * a.W : a.dims[i - a.n_cross] * a.dims[i - a.n_cross + 1];
  };
  auto woff = [&](int i) {  // float offset of layer i's W^T (each rounded up to 4 floats: 16-byte aligned)
    int o = 0;
    for (int j = 0; j < i; ++j) o += (wn(j) + 3) & ~3;
    return o;
  };
  if (threadIdx.x == 0) {
    for (int l = 0; l < n_layers; ++l) ptx::mbar_init(&wbar[l], 1);
    ptx::fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int l = 0; l < n_layers; ++l) {
      const uint32_t bytes = (uint32_t)(wn(l) * 4) & ~15u;
      ptx::mbar_arrive_expect_tx(&wbar[l], bytes);
      if (bytes)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         ptx::smem_u32(wbase + woff(l))),
                     "l"(wt(l)), "r"(bytes), "r"(ptx::smem_u32(&wbar[l]))
                     : "memory");
    }
  }
  for (int l = 0; l < n_layers; ++l) {  // the < 16-byte tails, plain loads
    const int n = wn(l), t0 = (int)(((uint32_t)(n * 4) & ~15u) >> 2);
    for (int i = t0 + threadIdx.x; i < n; i += blockDim.x) wbase[woff(l) + i] = __ldg(wt(l) + i);
  }
  const int row0 = blockIdx.x * R;
  for (int i = threadIdx.x; i < R * a.W; i += blockDim.x) {
    const int r = i / a.W, c = i - r * a.W;
    const float v = (row0 + r < B) ? a.x0[(int64_t)(row0 + r) * a.x0_ld + c] : 0.f;
    x0s[r * ld + c] = v;
    bufA[r * ld + c] = v;
  }
  float* cur = bufA;
  float* nxt = bufB;
  for (int l = 0; l < n_layers; ++l) {
    ptx::mbar_wait(&wbar[l], 0);  // layer l's weights landed
    __syncthreads();              // the tails and the activations are visible
    const float* w = wbase + woff(l);
    if (l < a.n_cross) {
      layer4<true>(cur, a.W, nxt, a.W, ld, w, a.bias[l], x0s);
    } else {
      const int i = l - a.n_cross;
      layer4<false>(cur, a.dims[i], nxt, a.dims[i + 1], ld, w, a.mb[i], nullptr);
    }
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
    if (lane == 0 && row0 + r < B) scores[row0 + r] = sigmoid_f32(s + __ldg(a.head_b));
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
  wmax = (wmax + 3) & ~(size_t)3;  // keeps the second buffer 16-byte aligned
  // all layers resident when they fit
  size_t wall = 0;
  for (int i = 0; i < a.n_cross; ++i) wall += ((size_t)a.W * a.W + 3) & ~(size_t)3;
  for (int i = 0; i < a.n_mlp; ++i) wall += ((size_t)a.dims[i] * a.dims[i + 1] + 3) & ~(size_t)3;
  const size_t smem_res = ((size_t)3 * R * ld + wall) * sizeof(float);
  if (smem_res <= 220 * 1024 && a.n_cross + a.n_mlp <= kMaxLayers) {
    static size_t attr_res = 0;
    if (smem_res > 48 * 1024 && smem_res > attr_res) {
      cudaError_t e = cudaFuncSetAttribute(dense_f32_resident_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)smem_res);
      if (e != cudaSuccess) return e;
      attr_res = smem_res;
    }
    dense_f32_resident_kernel<<<(a.B + R - 1) / R, 256, smem_res, s>>>(a, ld);
    return cudaGetLastError();
  }
  const size_t smem = ((size_t)3 * R * ld + 2 * wmax) * sizeof(float);
  if (smem > 220 * 1024) return cudaErrorInvalidValue;
  static size_t attr_set = 0;
  if (smem > 48 * 1024 && smem > attr_set) {
    cudaError_t e = cudaFuncSetAttribute(dense_f32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr_set = smem;
  }
  dense_f32_kernel<<<(a.B + R - 1) / R, 256, smem, s>>>(a, ld, (int)wmax);
  return cudaGetLastError();
}

}  // namespace cvr
