// embed.cu -- K1 embedding-bag gather + sum-pool, K2 dense normalisation + concat, and the
// sharded-mode unpack.
//
// S2 (§2.1; BASELINE.json north star (a)):
//     p[b, t, :] = sum_{j = off[t*B+b]}^{off[t*B+b+1]-1} E_t[idx[j], :]
// fp32 accumulation in index order, stored in the x0 dtype.  HBM-bound gather, no tensor
// cores: a group of LPR = d*sizeof(row elt)/16 lanes owns one bag, each lane owns 16 bytes of
// the row (one 128-bit ld.global.nc per row); latency is hidden by occupancy (64 warps/SM, 32
// registers) rather than by deep per-lane unrolling (measured fastest).  Consecutive
// groups take consecutive bags of the same table (table-major CSR), so Zipf-hot rows of a
// table are re-read from L2 by neighbouring warps.
//
// S3 ("normal standardization"): x0[b, T*d + f] = (x[b,f] - mu_f) / sigma_f,
// computed in fp32 with a correctly rounded division, by extra CTAs of the same grid.
//
// Feature front end, fused into the same gather: in keys mode each bag element is a
// raw 64-bit key, hashed on the fly -- FNV-1a 64 over its 8 big-endian bytes, modulo the table's vocab,
// the MISSING key (all ones) mapping to the `unseen' row vocab --
// and tables flagged `mean' divide the fp32 sum by the bag length (PAPER.md:97 average pooling of text
// n-grams; sequences); empty bags pool to 0 in both modes.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "cvr_kernels.cuh"
#include "cvr_ptx.cuh"

namespace cvr {
namespace {

template <typename T>
struct InTraits;
template <>
struct InTraits<float> {
  static constexpr int EPL = 4;
  __device__ static void add(float* acc, const uint4& v) {
    acc[0] += __uint_as_float(v.x);
    acc[1] += __uint_as_float(v.y);
    acc[2] += __uint_as_float(v.z);
    acc[3] += __uint_as_float(v.w);
  }
};
template <>
struct InTraits<__nv_bfloat16> {
  static constexpr int EPL = 8;
  __device__ static void add(float* acc, const uint4& v) {
    acc[0] += ptx::bf16_lo(v.x);
    acc[1] += ptx::bf16_hi(v.x);
    acc[2] += ptx::bf16_lo(v.y);
    acc[3] += ptx::bf16_hi(v.y);
    acc[4] += ptx::bf16_lo(v.z);
    acc[5] += ptx::bf16_hi(v.z);
    acc[6] += ptx::bf16_lo(v.w);
    acc[7] += ptx::bf16_hi(v.w);
  }
};
template <>
struct InTraits<__half> {
  static constexpr int EPL = 8;
  __device__ static void add(float* acc, const uint4& v) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float2 f = __half22float2(*reinterpret_cast<const __half2*>(&w[i]));
      acc[2 * i] += f.x;
      acc[2 * i + 1] += f.y;
    }
  }
};

template <int EPL>
__device__ __forceinline__ void store_out(float* dst, const float* acc) {
#pragma unroll
  for (int i = 0; i < EPL; i += 4)
    *reinterpret_cast<float4*>(dst + i) = make_float4(acc[i], acc[i + 1], acc[i + 2], acc[i + 3]);
}
template <int EPL>
__device__ __forceinline__ void store_out(__nv_bfloat16* dst, const float* acc) {
  if constexpr (EPL == 8) {
    uint4 v = make_uint4(ptx::pack_bf16(acc[0], acc[1]), ptx::pack_bf16(acc[2], acc[3]),
                         ptx::pack_bf16(acc[4], acc[5]), ptx::pack_bf16(acc[6], acc[7]));
    *reinterpret_cast<uint4*>(dst) = v;
  } else {
    uint2 v = make_uint2(ptx::pack_bf16(acc[0], acc[1]), ptx::pack_bf16(acc[2], acc[3]));
    *reinterpret_cast<uint2*>(dst) = v;
  }
}

__device__ __forceinline__ void store_scalar(float* p, float v) { *p = v; }
__device__ __forceinline__ void store_scalar(__nv_bfloat16* p, float v) { *p = __float2bfloat16_rn(v); }

template <typename TOut>
__device__ void dense_part(const EmbedArgs& a, const float* dense, int Bd, int blk, int nblk) {
  const int64_t ncols = a.pad_col1 - a.dense_col0;
  const int64_t total = (int64_t)Bd * ncols;
  TOut* x0 = reinterpret_cast<TOut*>(a.x0);
  for (int64_t i = (int64_t)blk * blockDim.x + threadIdx.x; i < total; i += (int64_t)nblk * blockDim.x) {
    const int64_t r = i / ncols;
    const int c = (int)(i - r * ncols);
    float v = 0.f;
    if (c < a.F) v = __fdiv_rn(__ldg(dense + r * a.F + c) - __ldg(a.mean + c), __ldg(a.sigma + c));
    store_scalar(x0 + r * a.x0_ld + a.dense_col0 + c, v);
  }
}

__device__ __forceinline__ int64_t hashed_row(uint64_t key, int64_t vocab, uint64_t magic) {
  if (key == ~0ull) return vocab;  // MISSING -> unseen row
  uint64_t h = 0xCBF29CE484222325ull;
#pragma unroll
  for (int i = 7; i >= 0; --i) {  // big-endian byte order
    h ^= (key >> (8 * i)) & 0xFFull;
    h *= 0x100000001B3ull;
  }
  // h mod vocab by a precomputed reciprocal: the quotient estimate is low by at most 2
  uint64_t r = h - __umul64hi(h, magic) * (uint64_t)vocab;
  while (r >= (uint64_t)vocab) r -= (uint64_t)vocab;
  return (int64_t)r;
}

// NA: row loads that do not allocate in L1 (rows of <= 128 B, see launch_t)
template <typename TIn, typename TOut, int LPR, int MINB, bool KEYS, bool NA = false>
__global__ void __launch_bounds__(256, MINB) embed_bag_kernel(const EmbedArgs a, int n_embed_blocks) {
  // this batch's inputs: from the executor's per-call block (one graph serves every batch), else the launch's
  const int32_t* indices = a.indices;
  const uint64_t* keys = a.keys;
  const int32_t* offsets = a.offsets;
  const float* dense = a.dense;
  int64_t nnz = a.nnz;
  int B = a.B, Bd = a.Bd;
  if (a.call) {
    indices = a.call->indices;
    keys = a.call->keys;
    offsets = a.call->offsets;
    dense = a.call->dense;
    nnz = a.call->nnz;
    B = Bd = a.call->B;
  }
  if ((int)blockIdx.x >= n_embed_blocks) {
    dense_part<TOut>(a, dense, Bd, blockIdx.x - n_embed_blocks, gridDim.x - n_embed_blocks);
    return;
  }
  constexpr int EPL = InTraits<TIn>::EPL;
  const int sub = threadIdx.x & (LPR - 1);
  const int64_t n_bags = (int64_t)a.T * B;
  const int64_t stride = (int64_t)n_embed_blocks * blockDim.x / LPR;
  for (int64_t bag = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / LPR; bag < n_bags; bag += stride) {
    const int t = (int)(bag / B);
    const int b = (int)(bag - (int64_t)t * B);
    const int64_t start = __ldg(offsets + bag);
    const int64_t end = __ldg(offsets + bag + 1);
    const TableDesc td = a.tables[t];
    float acc[EPL];
#pragma unroll
    for (int e = 0; e < EPL; ++e) acc[e] = 0.f;
    bool bad = start < 0 || end < start || end > nnz;
    if (!bad) {
      const uint8_t* colbase = td.base + sub * 16;
      if constexpr (KEYS) {
        // each lane of the group fetches (keys: and hashes) one element of the next LPR -- one coalesced
        // load per group -- then the row ids are broadcast in turn, two row loads in flight per lane
        const unsigned gmask = (LPR == 32) ? 0xffffffffu : (((1u << LPR) - 1) << (threadIdx.x & 31 & ~(LPR - 1)));
        for (int64_t j0 = start; j0 < end; j0 += LPR) {
          const int64_t jj = j0 + sub;
          int64_t my = 0;
          if (jj < end) {
            my = hashed_row(__ldg(keys + jj), td.vocab, td.magic);
          }
          bad |= jj < end && (my < 0 || my >= td.rows);
          bad = __any_sync(gmask, bad);
          if (bad) break;
          const int cnt = (int)((end - j0) < LPR ? (end - j0) : LPR);
          int u = 0;
          for (; u + 1 < cnt; u += 2) {
            const int64_t r0 = __shfl_sync(gmask, my, u, LPR), r1 = __shfl_sync(gmask, my, u + 1, LPR);
            const uint4 v0 = ptx::ld_nc_v4(colbase + r0 * td.stride), v1 = ptx::ld_nc_v4(colbase + r1 * td.stride);
            InTraits<TIn>::add(acc, v0);
            InTraits<TIn>::add(acc, v1);
          }
          if (u < cnt) {
            const int64_t r0 = __shfl_sync(gmask, my, u, LPR);
            InTraits<TIn>::add(acc, ptx::ld_nc_v4(colbase + r0 * td.stride));
          }
        }
      } else
      for (int64_t j = start; j < end; ++j) {  // one row load in flight per lane (occupancy hides latency)
        const int64_t idx = (int64_t)__ldg(indices + j);
        bad |= idx < 0 || idx >= td.rows;
        if (bad) break;  // uniform within the group: every lane read the same index
        uint4 v;
        if constexpr (NA) v = ptx::ld_nc_na_v4(colbase + idx * td.stride);
        else v = ptx::ld_nc_v4(colbase + idx * td.stride);
        InTraits<TIn>::add(acc, v);
      }
    }
    if (bad) {
#pragma unroll
      for (int e = 0; e < EPL; ++e) acc[e] = 0.f;
      if (sub == 0) atomicOr(a.flag, 1);
    } else if (td.mean && end > start) {
      const float L = (float)(end - start);
#pragma unroll
      for (int e = 0; e < EPL; ++e) acc[e] = __fdiv_rn(acc[e], L);
    }
    TOut* dst;
    if (a.peer_x0) {  // V3: straight into the owner rank's canonical x0 (peer memory over NVLink)
      const int owner = b / a.Bl, bl = b - owner * a.Bl;
      dst = reinterpret_cast<TOut*>(a.peer_x0[owner]) + (int64_t)bl * a.x0_ld +
            (int64_t)(t * a.world + a.rank) * a.d + sub * EPL;
    } else {
      dst = reinterpret_cast<TOut*>(a.out) + (int64_t)b * a.out_ld + (int64_t)t * a.out_tstride + sub * EPL;
    }
    store_out<EPL>(dst, acc);
  }
}

template <typename TIn, typename TOut, int LPR>
cudaError_t launch_t(const EmbedArgs& a, int num_sms, cudaStream_t s) {
  const int threads = 256;
  // (executor graphs: a.B = a.Bd = max_batch here; the kernel reads the batch's B from a.call)
  const int64_t n_bags = (int64_t)a.T * a.B;
  // one bag per lane group, no grid-stride loop at full size: short-lived CTAs let the block scheduler
  // interleave the concurrently running dense-stage GEMM CTAs (higher-priority stream) as embed CTAs retire
  int64_t nbE = (n_bags * LPR + threads - 1) / threads;
  const int64_t capE = (int64_t)num_sms * (a.blocks_per_sm > 0 ? a.blocks_per_sm : 64);
  if (nbE > capE) nbE = capE;
  int64_t nbD = 0;
  if (a.x0 && a.Bd > 0 && a.pad_col1 > a.dense_col0) {
    const int64_t total = (int64_t)a.Bd * (a.pad_col1 - a.dense_col0);
    nbD = (total + threads - 1) / threads;
    if (nbD > num_sms) nbD = num_sms;
  }
  if (nbE + nbD == 0) return cudaSuccess;
  if (a.peer_x0 && a.keys) return cudaErrorInvalidValue;  // V3 uses the row-id kernel
  if (a.keys)
    embed_bag_kernel<TIn, TOut, LPR, 8, true><<<(unsigned)(nbE + nbD), threads, 0, s>>>(a, (int)nbE);
  else if (LPR <= 8)
    // rows of <= 128 B (one line each): row loads skip L1 allocation.  Measured on B200 (round 1): c2 (128-B bf16
    // rows) 20.3 -> 18.5 us; wider rows keep L1 allocation (c3-S 256-B rows 1.83 vs 2.00 ms, c4 512-B rows 187 vs
    // 203 us without it).  One row load in flight per lane at full occupancy (32 registers, 64 warps/SM) beat
    // deeper per-lane unrolling at lower occupancy (18.5 vs 24.6 us for 4 rows in flight at 32 warps/SM).
    embed_bag_kernel<TIn, TOut, LPR, 8, false, true><<<(unsigned)(nbE + nbD), threads, 0, s>>>(a, (int)nbE);
  else
    embed_bag_kernel<TIn, TOut, LPR, 8, false><<<(unsigned)(nbE + nbD), threads, 0, s>>>(a, (int)nbE);
  return cudaGetLastError();
}

template <typename TIn, typename TOut>
cudaError_t launch_lpr(const EmbedArgs& a, int num_sms, cudaStream_t s) {
  const int elt = a.emb_dtype == F32 ? 4 : 2;
  switch (a.d * elt / 16) {
    case 2: return launch_t<TIn, TOut, 2>(a, num_sms, s);
    case 4: return launch_t<TIn, TOut, 4>(a, num_sms, s);
    case 8: return launch_t<TIn, TOut, 8>(a, num_sms, s);
    case 16: return launch_t<TIn, TOut, 16>(a, num_sms, s);
    case 32: return launch_t<TIn, TOut, 32>(a, num_sms, s);
    default: return cudaErrorInvalidValue;
  }
}

__global__ void unpack_kernel(const uint4* __restrict__ recv, uint8_t* __restrict__ x0, int64_t x0_ld_bytes, int N,
                              int Bl, int Tpad, int T, int chunks_per_row, int row_bytes) {
  const int64_t total = (int64_t)N * Bl * Tpad * chunks_per_row;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t q = i;
    const int c = (int)(q % chunks_per_row);
    q /= chunks_per_row;
    const int slot = (int)(q % Tpad);
    q /= Tpad;
    const int b = (int)(q % Bl);
    const int src = (int)(q / Bl);
    const int t = slot * N + src;  // round-robin table placement, t -> rank t % N, slot t / N
    if (t >= T) continue;
    *reinterpret_cast<uint4*>(x0 + (int64_t)b * x0_ld_bytes + (int64_t)t * row_bytes + c * 16) = recv[i];
  }
}

__global__ void set_call_kernel(const CallArgs v, CallArgs* dst) {
  if (threadIdx.x == 0) *dst = v;
}

__global__ void peer_signal_kernel(uint32_t* const* __restrict__ peer_flags, int world, int rank, uint32_t epoch) {
  // the gather kernel before us on this stream has completed; make its peer stores visible system-wide
  // before publishing the epoch
  __threadfence_system();
  for (int d = threadIdx.x; d < world; d += blockDim.x) {
    uint32_t* f = peer_flags[d] + rank;
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(f), "r"(epoch) : "memory");
  }
}

__global__ void peer_wait_kernel(const uint32_t* __restrict__ flags, int world, uint32_t epoch) {
  for (int src = threadIdx.x; src < world; src += blockDim.x) {
    uint32_t v;
    do {
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flags + src) : "memory");
    } while ((int32_t)(v - epoch) < 0);
  }
  __syncthreads();
  __threadfence_system();
}

}  // namespace

cudaError_t launch_set_call(const CallArgs& v, CallArgs* d_call, cudaStream_t s) {
  set_call_kernel<<<1, 32, 0, s>>>(v, d_call);
  return cudaGetLastError();
}

cudaError_t launch_peer_signal(uint32_t* const* d_peer_flags, int world, int rank, uint32_t epoch, cudaStream_t s) {
  peer_signal_kernel<<<1, 32, 0, s>>>(d_peer_flags, world, rank, epoch);
  return cudaGetLastError();
}

cudaError_t launch_peer_wait(const uint32_t* d_flags, int world, uint32_t epoch, cudaStream_t s) {
  peer_wait_kernel<<<1, 32, 0, s>>>(d_flags, world, epoch);
  return cudaGetLastError();
}

cudaError_t launch_embed(const EmbedArgs& a, int num_sms, cudaStream_t s) {
  if (a.emb_dtype == F32 && a.out_dtype == F32) return launch_lpr<float, float>(a, num_sms, s);
  if (a.emb_dtype == F32 && a.out_dtype == BF16) return launch_lpr<float, __nv_bfloat16>(a, num_sms, s);
  if (a.emb_dtype == BF16 && a.out_dtype == BF16) return launch_lpr<__nv_bfloat16, __nv_bfloat16>(a, num_sms, s);
  if (a.emb_dtype == BF16 && a.out_dtype == F32) return launch_lpr<__nv_bfloat16, float>(a, num_sms, s);
  if (a.emb_dtype == F16 && a.out_dtype == BF16) return launch_lpr<__half, __nv_bfloat16>(a, num_sms, s);
  if (a.emb_dtype == F16 && a.out_dtype == F32) return launch_lpr<__half, float>(a, num_sms, s);
  return cudaErrorInvalidValue;
}

cudaError_t launch_unpack(const void* recv, void* x0, int64_t x0_ld, int N, int Bl, int Tpad, int T, int d,
                          int dtype, cudaStream_t s) {
  const int elt = dtype == F32 ? 4 : 2;
  const int row_bytes = d * elt;
  if (row_bytes % 16) return cudaErrorInvalidValue;
  const int cpr = row_bytes / 16;
  const int64_t total = (int64_t)N * Bl * Tpad * cpr;
  if (total == 0) return cudaSuccess;
  int64_t blocks = (total + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  unpack_kernel<<<(unsigned)blocks, 256, 0, s>>>(reinterpret_cast<const uint4*>(recv),
                                                   reinterpret_cast<uint8_t*>(x0), x0_ld * elt, N, Bl, Tpad, T, cpr,
                                                   row_bytes);
  return cudaGetLastError();
}

}  // namespace cvr
