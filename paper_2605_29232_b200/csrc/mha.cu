// mha.cu -- K7: multi-head self-attention over the 64 "global tokens" of each example (config 4,
// SURVEY.md §8(a) S5', reading A20; "Transformers ... self-attention", global tokens
// PAPER.md:245), plus the finaliser of the split head (EPI_HEAD_PARTIAL).
//
//   per example b and head h (dh = 64):  O_h = softmax(Q_h K_h^T / sqrt(dh)) V_h     (S = 64 tokens)
//
// S = Q K^T and O = P V run on the tensor cores as mma.sync m16n8k16 bf16 with fp32 accumulation; the
// 64x64 score tile of a head never leaves registers: row max / exp / sum in fp32 across the 4 lanes
// sharing a row, P rounded to bf16 as the second MMA's A operand (A26: P is a bf16 MMA operand).  The
// whole problem per (example, head) is 64x64x64 twice, far below a tcgen05 tile (M >= 64 per CTA with
// TMEM setup per tile), so the warp-level MMA is the right size here.
#include <cuda_bf16.h>

#include "cvr_attn.cuh"
#include "cvr_kernels.cuh"
#include "cvr_ptx.cuh"

namespace cvr {
namespace {

constexpr int S = 64;        // tokens
constexpr int DH = 64;       // head dim

// v2: one CTA per (example, head), 4 warps x 16 query rows.  Q, K, V of the head are copied with
// cp.async (16-byte, no register staging) into padded shared memory (row stride 72 elements: every
// ldmatrix phase hits 32 distinct banks); operands are fetched with ldmatrix (.trans for V, so V needs no
// transposed copy); 8 CTAs fit per SM (27 KB each) so the copies of some CTAs overlap the MMAs of others.
constexpr int LD2 = 72;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(ptx::smem_u32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}
template <int H>
__global__ void __launch_bounds__(128) mha64_v2_kernel(const __nv_bfloat16* __restrict__ qkv, __nv_bfloat16* __restrict__ out,
                                                       int out_ld, const CallArgs* call) {
  constexpr int D = H * DH;
  __shared__ __align__(128) __nv_bfloat16 Qs[S * LD2];
  __shared__ __align__(128) __nv_bfloat16 Ks[S * LD2];
  __shared__ __align__(128) __nv_bfloat16 Vs[S * LD2];
  const int b = blockIdx.x / H, h = blockIdx.x % H;
  if (call && b >= call->B) return;  // executor graphs: grid sized for max_batch
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const __nv_bfloat16* src = qkv + (size_t)b * S * 3 * D + h * DH;
  // 3 x 64 rows x 8 chunks of 16 bytes
  for (int i = tid; i < 3 * S * 8; i += blockDim.x) {
    const int m = i / (S * 8), rem = i % (S * 8), tok = rem >> 3, ch = rem & 7;
    __nv_bfloat16* dst = (m == 0 ? Qs : m == 1 ? Ks : Vs) + tok * LD2 + ch * 8;
    cp_async16(dst, src + (size_t)tok * 3 * D + m * D + ch * 8);
  }
  cp_async_wait_all();
  __syncthreads();
  const int r0 = warp * 16;
  attn::rows16<LD2>(Qs, Ks, Vs, r0, lane);  // O rows r0..r0+15 now in Qs (cvr_attn.cuh)
  __nv_bfloat16* Os = Qs + r0 * LD2;
  __syncwarp();
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    const int row = p * 4 + (lane >> 3), ch = lane & 7;
    *reinterpret_cast<uint4*>(out + ((size_t)b * S + r0 + row) * out_ld + h * DH + ch * 8) =
        *reinterpret_cast<const uint4*>(Os + row * LD2 + ch * 8);
  }
}

__device__ __forceinline__ float sigmoid_f32(float z) {
  if (z >= 0.f) return 1.f / (1.f + expf(-z));
  const float e = expf(z);
  return e / (1.f + e);
}

__global__ void head_finalize_kernel(const float* __restrict__ part, int n_parts, float c, float* __restrict__ scores,
                                     int M, const CallArgs* call) {
  if (call) {  // executor graphs: this batch's rows and scores pointer
    M = call->B;
    scores = call->scores;
  }
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= M) return;
  float z = 0.f;
  for (int j = 0; j < n_parts; ++j) z += part[(size_t)m * n_parts + j];  // fixed order: batch invariant
  scores[m] = sigmoid_f32(z + c);
}

}  // namespace

cudaError_t launch_mha64(const __nv_bfloat16* qkv, __nv_bfloat16* out, int out_ld, int B, int n_heads, cudaStream_t s,
                         const CallArgs* call) {
  if (B <= 0) return cudaSuccess;
  if (n_heads != 4) return cudaErrorInvalidValue;
  if (out_ld % 8) return cudaErrorInvalidValue;
  mha64_v2_kernel<4><<<B * 4, 128, 0, s>>>(qkv, out, out_ld, call);
  return cudaGetLastError();
}

cudaError_t launch_head_finalize(const float* partial, int n_parts, float c, float* scores, int M, cudaStream_t s,
                                 const CallArgs* call) {
  if (M <= 0) return cudaSuccess;
  head_finalize_kernel<<<(M + 255) / 256, 256, 0, s>>>(partial, n_parts, c, scores, M, call);
  return cudaGetLastError();
}

}  // namespace cvr
