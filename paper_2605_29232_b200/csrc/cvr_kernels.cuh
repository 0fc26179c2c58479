// cvr_kernels.cuh -- internal launchers of the hot-path kernels (not part of the C ABI).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

namespace cvr {

enum DType { F32 = 0, BF16 = 1, F16 = 2 };

struct TableDesc {
  const uint8_t* base;  // row 0
  int64_t stride;       // bytes between rows
  int64_t rows;
  int64_t vocab;        // keys mode: hash modulus (row vocab = the `unseen' row); 0 = indices are row ids
  uint64_t magic;       // floor((2^64 - 1) / vocab): h mod vocab = h - umulhi(h, magic) * vocab (+ <= 2 fixes)
  int mean;             // 1: mean pooling (sum / bag length, empty -> 0); 0: sum pooling
};

// ---- per-call argument block of the executor (device memory, one per x0 slot) ---------------------------
// cvr_score / cvr_score_host replay ONE captured CUDA graph per (stage, slot) for every batch: the batch's
// pointers and row count live in this block, written on the embed stream right before the embed graph
// (launch_set_call), and every kernel of both stages reads them from here instead of its launch parameters
// (one graph per stage for every batch size <= max_batch, device-side row count).
struct CallArgs {
  const int32_t* indices;
  const uint64_t* keys;
  const int32_t* offsets;
  const float* dense;
  float* scores;
  int64_t nnz;
  int B;                     // rows of this batch (<= max_batch)
  int pad;
};
cudaError_t launch_set_call(const CallArgs& v, CallArgs* d_call, cudaStream_t s);

// ---- K1 + K2: embedding-bag sum-pool (+ dense normalisation) --------------------------------
struct EmbedArgs {
  const TableDesc* tables;   // device array [T_local]
  const int32_t* indices;
  const uint64_t* keys;      // keys mode (feature front end): raw 64-bit keys instead of indices
  const int32_t* offsets;    // [T_local * B + 1]
  int64_t nnz;
  int B;                     // bags per table (global batch in sharded mode)
  int T;                     // tables handled (T_local)
  int d;
  int emb_dtype, out_dtype;
  void* out;                 // pooled output base
  int64_t out_ld;            // elements between consecutive b
  int64_t out_tstride;       // elements between consecutive tables (column offset t*out_tstride)
  // dense normalisation (S3); skipped when F == 0 or dense == nullptr
  const float* dense;        // [Bd, F]
  int Bd;                    // rows of dense
  int F;
  const float* mean;         // [F]
  const float* sigma;        // [F] (floored at 1e-8 at load)
  void* x0;                  // x0 base for dense columns
  int64_t x0_ld;
  int64_t dense_col0;        // first dense column (T_total * d)
  int64_t pad_col0, pad_col1;  // zero columns [pad_col0, pad_col1) of x0 rows
  int* flag;                 // sticky error flag
  const CallArgs* call;      // executor graphs: indices / keys / offsets / nnz / B (= Bd) / dense come from here
                             // (B above then only sizes the grid: max_batch)
  int blocks_per_sm;         // grid cap (grid-stride): leaves registers for co-resident GEMM CTAs
  // fused exchange (V3): pooled rows go straight into the owner rank's canonical x0
  // through peer-mapped pointers: bag (t_local, b) -> peer_x0[b / Bl] row b % Bl, columns (t_local*world+rank)*d
  void* const* peer_x0;      // device array [world] of destination x0 bases ([Bl, x0_ld] each); null = off
  int world, rank, Bl;
};
// V3 handshake: after the fused gather, rank `rank` sets flags_of[dst][rank] = epoch on every destination
// (release, system scope); the dense stage of rank dst first waits until its own flags[src] >= epoch for all src.
cudaError_t launch_peer_signal(uint32_t* const* d_peer_flags, int world, int rank, uint32_t epoch, cudaStream_t s);
cudaError_t launch_peer_wait(const uint32_t* d_flags, int world, uint32_t epoch, cudaStream_t s);
cudaError_t launch_embed(const EmbedArgs& a, int num_sms, cudaStream_t s);

// unpack received shard chunks [src][b_local][t_slot][d] into canonical x0 columns
cudaError_t launch_unpack(const void* recv, void* x0, int64_t x0_ld, int N, int Bl, int Tpad, int T, int d,
                          int dtype, cudaStream_t s);

// ---- K3: fp32 fused DCN-full forward (config 1) ------------------------------------------------
constexpr int kMaxLayers = 8;
struct DenseF32Args {
  const float* x0;
  int64_t x0_ld;
  int B, W;
  int n_cross;
  const float* WT[kMaxLayers];    // W_l^T [W][W] (in-major, repacked at load)
  const float* bias[kMaxLayers];  // b_l [W]
  int n_mlp;
  int dims[kMaxLayers + 1];       // W, h_1, ..., h_n
  const float* MT[kMaxLayers];    // M_i^T [in][out]
  const float* mb[kMaxLayers];    // c_i [out]
  const float* head_w;            // [h_n]
  const float* head_b;            // [1]
  float* scores;
  const CallArgs* call;           // executor graphs: B and scores from the call block (B above sizes the grid)
};
cudaError_t launch_dense_f32(const DenseF32Args& a, cudaStream_t s);

// ---- config 4: FFN1 + out-projection + FFN2 + branch-sum LN in one tcgen05 kernel (ffn_fused.cu) ----------
struct FfnArgs {
  const CUtensorMap *tmX, *tmO;          // X tokens [M, D] and cat [M, D + F] (O = its first D columns), box 64 x 128
  const CUtensorMap *tmW1;               // W1 [F, D], box 64 x 128
  const CUtensorMap *tmW2, *tmWo;        // [Wo | W2] [D, D + F]: box 64 x 256 (W2 part), 64 x 128 (Wo halves)
  const CUtensorMap *tmS;                // S fp32 [M, D] (the DCN branch), box 32 x 32
  const CUtensorMap *tmOut;              // X' bf16 [M, D], store box 64 x 32
  const float *b1, *bcat, *gamma, *beta; // b1 [F]; bo + b2 [D]; LN affine [D]
  int M, F, D, m_mult, num_sms;
  bool pdl;
  const CallArgs* call;                  // executor graphs: tokens = call->B * m_mult
};
cudaError_t launch_ffn_fused(const FfnArgs& g, cudaStream_t s);

// ---- K4: tcgen05 bf16 GEMM with fused epilogues --------------------------------------------------
enum Epi {
  EPI_STORE = 0,         // bf16 C
  EPI_BIAS_RELU = 1,     // bf16 ReLU(C + b)
  EPI_CROSS = 2,         // bf16 x0 * (C + b) + x_l
  EPI_HEAD = 3,          // fp32 sigmoid(ReLU(C + b) . m + c)            (BN == N)
  EPI_BIAS = 4,          // bf16 C + b
  EPI_CROSS_F32 = 5,     // fp32 x0 * (C + b) + x_l                      (ensemble DCN branch)
  EPI_BIAS_ADD_F32 = 6,  // fp32 C + b + in_f32                          (ensemble MHA out-proj)
  EPI_SUM_LN = 7,        // bf16 LN_row(C + b + in_f32) * gamma + beta   (ensemble FFN2 + LN, BN == N)
  EPI_HEAD_PARTIAL = 8,  // fp32 partial[m][tile] = ReLU(C + b) . m over the tile's columns
  EPI_MASK = 9,          // bf16 (C + b) * x_l: MaskNet block, mask applied to x_l (tmXl), no residual
  EPI_ATTN = 10,         // config 4: the 128 x 192 tile [q_h | k_h | v_h] (+ b) of 2 examples' tokens -> attention of
                         // head h = N tile -> O (bf16) at out_bf16[token, 64 h ..] (row stride ld_x); BN = 192
  EPI_ATTN_TC = 11       // the same on tcgen05: S = Q K^T and O = P V as UMMAs into the drained accumulator's TMEM
                         // columns, softmax thread-per-row from TMEM; O TMA-stored through tmOut (box {64, 128})
};

struct GemmArgs {
  const CUtensorMap* tmA;    // A [M, K] bf16, box {64, 128}
  const CUtensorMap* tmB;    // B [N, K] bf16, box {64, BN}
  const CUtensorMap* tmOut;  // C [M, N] bf16, box {64, 32} (not EPI_HEAD)
  const CUtensorMap* tmX0;   // EPI_CROSS: x0 [M, N], box {64, 128}
  const CUtensorMap* tmXl;   // EPI_CROSS: x_l [M, N], box {64, 128}
  const float* bias;         // fp32 [N] (not EPI_STORE)
  const float* head_w;       // EPI_HEAD fp32 [N]
  float head_b;
  float* scores;             // EPI_HEAD fp32 [M]
  float* out_f32;            // EPI_CROSS_F32 / EPI_BIAS_ADD_F32: fp32 [M, ld_f32]
  int64_t ld_f32;
  const float* in_f32;       // EPI_BIAS_ADD_F32 / EPI_SUM_LN: fp32 [M, ld_in] (may alias out_f32)
  int64_t ld_in;
  const float* gamma;        // EPI_SUM_LN [N]
  const float* beta;         // EPI_SUM_LN [N]
  float* partial;            // EPI_HEAD_PARTIAL [M, N / BN]
  __nv_bfloat16* out_bf16;   // EPI_ATTN: O [M, ld_x] bf16 (written with plain stores)
  int64_t ld_x;
  int M, N, K, BN;
  Epi epi;
  int num_sms;
  bool pdl;                  // launch with programmatic stream serialization
  bool cta_pair;             // 2-CTA (cta_group::2) tiles of 256 rows; B box = BN/2 rows
  bool epw1;                 // one epilogue warp per TMEM quadrant (several tiles per CTA; see Cfg::EPW)
  int group_n;               // EPI_MASK grouped over branches: N tiles of group g = n / group_n read A columns
                             // [g K, (g + 1) K) and x_l columns n - g group_n (0 = off)
  bool no_prefetch_b;        // do not issue the first ring stages' B (weight) loads before griddepcontrol.wait
  const CallArgs* call;      // executor graphs: M = call->B * m_mult and scores = call->scores are read on the
  int m_mult;                // device (M above then sizes the grid for max_batch; m_mult = rows per example)
  unsigned long long* dbg;   // optional per-CTA timeline [grid][8] (%globaltimer ns): entry, deps ready,
                             // first stage landed, last MMA issued, first accumulator, epilogue done, exit
};

// C[M, N] = epi(A[M, K] . B[N, K]^T).  K % 64 == 0, N % BN == 0, BN in {64, 128, 256};
// EPI_HEAD / EPI_SUM_LN need BN == N.  Persistent: grid = min(tiles, num_sms).
cudaError_t launch_gemm_bf16(const GemmArgs& g, cudaStream_t s);

// ---- K7: multi-head self-attention over the 64 tokens of each example (config 4) ------------------
// qkv [B*S, 3*D] bf16 (Q | K | V, head h at columns h*64 of each), out [B*S, D] bf16; S = 64, dh = 64.
cudaError_t launch_mha64(const __nv_bfloat16* qkv, __nv_bfloat16* out, int out_ld, int B, int n_heads, cudaStream_t s,
                         const CallArgs* call = nullptr);
// scores[m] = sigmoid(sum_j partial[m][j] + c), j in fixed order (EPI_HEAD_PARTIAL finaliser)
cudaError_t launch_head_finalize(const float* partial, int n_parts, float c, float* scores, int M, cudaStream_t s,
                                 const CallArgs* call = nullptr);

// host: encode a 2-D bf16 K-major tensor map [rows, cols] (row stride ld elements) with box
// {64, box_rows} and 128-byte swizzle.
// fp32 [rows, cols] (row stride ld elements), box {32 columns, 32 rows}, 128-byte swizzle: the staged fp32 epilogue
// stores (EPI_CROSS_F32)
int encode_tmap_f32_store(CUtensorMap* tm, const void* ptr, int64_t rows, int64_t cols, int64_t ld, const char** err);
int encode_tmap_bf16(CUtensorMap* tm, const void* ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows,
                     const char** err);

}  // namespace cvr
