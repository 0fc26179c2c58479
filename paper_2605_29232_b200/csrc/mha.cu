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

#include "cvr_kernels.cuh"
#include "cvr_ptx.cuh"

namespace cvr {
namespace {

constexpr int S = 64;        // tokens
constexpr int DH = 64;       // head dim

__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

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
__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(ptx::smem_u32(p)));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(ptx::smem_u32(p)));
}

template <int H>
__global__ void __launch_bounds__(128) mha64_v2_kernel(const __nv_bfloat16* __restrict__ qkv, __nv_bfloat16* __restrict__ out,
                                                       int out_ld) {
  constexpr int D = H * DH;
  __shared__ __align__(128) __nv_bfloat16 Qs[S * LD2];
  __shared__ __align__(128) __nv_bfloat16 Ks[S * LD2];
  __shared__ __align__(128) __nv_bfloat16 Vs[S * LD2];
  const int b = blockIdx.x / H, h = blockIdx.x % H;
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
  const int g = lane >> 2, t = lane & 3;
  const int r0 = warp * 16;
  // ---- S = Q K^T (16 rows x 64 keys)
  float sc[8][4];
#pragma unroll
  for (int nt = 0; nt < 8; ++nt) sc[nt][0] = sc[nt][1] = sc[nt][2] = sc[nt][3] = 0.f;
#pragma unroll
  for (int ks = 0; ks < DH / 16; ++ks) {
    uint32_t a[4];
    ldsm_x4(a, Qs + (r0 + (lane & 7) + ((lane >> 3) & 1) * 8) * LD2 + ks * 16 + (lane >> 4) * 8);
#pragma unroll
    for (int np = 0; np < 4; ++np) {  // two 8-key n-tiles per ldmatrix.x4
      uint32_t bq[4];
      ldsm_x4(bq, Ks + (np * 16 + (lane & 7) + (lane >> 4) * 8) * LD2 + ks * 16 + ((lane >> 3) & 1) * 8);
      mma16816(sc[2 * np], a, bq[0], bq[1]);
      mma16816(sc[2 * np + 1], a, bq[2], bq[3]);
    }
  }
  // ---- softmax over 64 keys for rows g and g+8 (scale 1/8 exact), fp32
  float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
  for (int nt = 0; nt < 8; ++nt) {
#pragma unroll
    for (int e = 0; e < 4; ++e) sc[nt][e] *= 0.125f;
    mx0 = fmaxf(mx0, fmaxf(sc[nt][0], sc[nt][1]));
    mx1 = fmaxf(mx1, fmaxf(sc[nt][2], sc[nt][3]));
  }
#pragma unroll
  for (int o = 1; o <= 2; o <<= 1) {
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, o));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, o));
  }
  float s0 = 0.f, s1 = 0.f;
#pragma unroll
  for (int nt = 0; nt < 8; ++nt) {
    sc[nt][0] = expf(sc[nt][0] - mx0);
    sc[nt][1] = expf(sc[nt][1] - mx0);
    sc[nt][2] = expf(sc[nt][2] - mx1);
    sc[nt][3] = expf(sc[nt][3] - mx1);
    s0 += sc[nt][0] + sc[nt][1];
    s1 += sc[nt][2] + sc[nt][3];
  }
#pragma unroll
  for (int o = 1; o <= 2; o <<= 1) {
    s0 += __shfl_xor_sync(0xffffffffu, s0, o);
    s1 += __shfl_xor_sync(0xffffffffu, s1, o);
  }
  const float i0 = 1.f / s0, i1 = 1.f / s1;
  // ---- O = P V (P re-used from the S fragments as bf16 A operands; V via ldmatrix.trans)
  float oc[8][4];
#pragma unroll
  for (int nt = 0; nt < 8; ++nt) oc[nt][0] = oc[nt][1] = oc[nt][2] = oc[nt][3] = 0.f;
#pragma unroll
  for (int kk = 0; kk < S / 16; ++kk) {
    uint32_t a[4];
    a[0] = ptx::pack_bf16(sc[2 * kk][0] * i0, sc[2 * kk][1] * i0);
    a[1] = ptx::pack_bf16(sc[2 * kk][2] * i1, sc[2 * kk][3] * i1);
    a[2] = ptx::pack_bf16(sc[2 * kk + 1][0] * i0, sc[2 * kk + 1][1] * i0);
    a[3] = ptx::pack_bf16(sc[2 * kk + 1][2] * i1, sc[2 * kk + 1][3] * i1);
#pragma unroll
    for (int np = 0; np < 4; ++np) {  // two 8-wide dh tiles per ldmatrix.x4.trans
      uint32_t bv[4];
      ldsm_x4_t(bv, Vs + (kk * 16 + (lane & 7) + ((lane >> 3) & 1) * 8) * LD2 + np * 16 + (lane >> 4) * 8);
      mma16816(oc[2 * np], a, bv[0], bv[1]);
      mma16816(oc[2 * np + 1], a, bv[2], bv[3]);
    }
  }
  // ---- stage O (this warp's 16 rows of Qs are free) and store 16-byte chunks coalesced
  __nv_bfloat16* Os = Qs + r0 * LD2;
#pragma unroll
  for (int nt = 0; nt < 8; ++nt) {
    *reinterpret_cast<uint32_t*>(Os + g * LD2 + nt * 8 + 2 * t) = ptx::pack_bf16(oc[nt][0], oc[nt][1]);
    *reinterpret_cast<uint32_t*>(Os + (g + 8) * LD2 + nt * 8 + 2 * t) = ptx::pack_bf16(oc[nt][2], oc[nt][3]);
  }
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
                                     int M) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= M) return;
  float z = 0.f;
  for (int j = 0; j < n_parts; ++j) z += part[(size_t)m * n_parts + j];  // fixed order: batch invariant
  scores[m] = sigmoid_f32(z + c);
}

}  // namespace

cudaError_t launch_mha64(const __nv_bfloat16* qkv, __nv_bfloat16* out, int out_ld, int B, int n_heads, cudaStream_t s) {
  if (B <= 0) return cudaSuccess;
  if (n_heads != 4) return cudaErrorInvalidValue;
  if (out_ld % 8) return cudaErrorInvalidValue;
  mha64_v2_kernel<4><<<B * 4, 128, 0, s>>>(qkv, out, out_ld);
  return cudaGetLastError();
}

cudaError_t launch_head_finalize(const float* partial, int n_parts, float c, float* scores, int M, cudaStream_t s) {
  if (M <= 0) return cudaSuccess;
  head_finalize_kernel<<<(M + 255) / 256, 256, 0, s>>>(partial, n_parts, c, scores, M);
  return cudaGetLastError();
}

}  // namespace cvr
