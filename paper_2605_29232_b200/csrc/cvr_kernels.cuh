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
  bool v2;                   // warp-batched variant (batched offsets / staged index runs)
  int variant;               // occupancy / unroll variant of the per-bag kernel (tuning)
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
};
cudaError_t launch_dense_f32(const DenseF32Args& a, cudaStream_t s);

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
  EPI_ATTN = 10          // config 4: the 128 x 192 tile [q_h | k_h | v_h] (+ b) of 2 examples' tokens -> attention of
                         // head h = N tile -> O (bf16) at out_bf16[token, 64 h ..] (row stride ld_x); BN = 192
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
  __nv_bfloat16* out_bf16;   // launch_gemm_splitk: C [M, ld_x] bf16 (written with plain stores)
  int64_t ld_x;
  int M, N, K, BN;
  Epi epi;
  int num_sms;
  bool pdl;                  // launch with programmatic stream serialization
  bool a_resident;           // K <= 256: keep the A block resident, contiguous tile runs per CTA
  bool cta_pair;             // 2-CTA (cta_group::2) tiles of 256 rows; B box = BN/2 rows
  bool epw1;                 // one epilogue warp per TMEM quadrant (several tiles per CTA; see Cfg::EPW)
  bool mb8;                  // clusters of 8 consecutive row blocks multicast the B tile (tmB box {64, BN/8})
  int group_n;               // EPI_MASK grouped over branches: N tiles of group g = n / group_n read A columns
                             // [g K, (g + 1) K) and x_l columns n - g group_n (0 = off)
  int cn;                    // 4: clusters of 4 CTAs along N multicast A (tmA box = {64, 32}); 0/1: off
  bool no_prefetch_b;        // do not issue the first ring stages' B (weight) loads before griddepcontrol.wait
  unsigned long long* dbg;   // optional per-CTA timeline [grid][8] (%globaltimer ns): entry, deps ready,
                             // first stage landed, last MMA issued, first accumulator, epilogue done, exit
};

// C[M, N] = epi(A[M, K] . B[N, K]^T).  K % 64 == 0, N % BN == 0, BN in {64, 128, 256};
// EPI_HEAD needs BN * cn == N.  Persistent: grid = min(tiles, num_sms).
cudaError_t launch_gemm_bf16(const GemmArgs& g, cudaStream_t s);

// t = A . B^T with N = 256 as one 128 x 256 tile per row block, K split over a cluster of 4 CTAs and reduced
// in DSMEM in a fixed order (gemm_splitk.cu).  Uses tmA (box {64, 128}), tmB (box {64, 256}), out_bf16 /
// ld_x (row stride of t), M, K, pdl.
cudaError_t launch_gemm_splitk(const GemmArgs& g, cudaStream_t s);

// ---- config 4: fused FFN + out-projection + branch-sum LayerNorm (ens_ffn.cu) ------------------------------
struct EnsFfnArgs {
  const CUtensorMap* tmX;    // x_l tokens [BT, D] box {64, 128}
  const CUtensorMap* tmO;    // MHA output O = cat[:, :D] (row stride D + F) box {64, 128}
  const CUtensorMap* tmW1;   // W1 [F, D] box {64, 128}
  const CUtensorMap* tmWc;   // [Wo | W2] [D, D + F] box {64, 256}
  const CUtensorMap* tmY;    // out tokens [BT, D] box {64, 32}
  const float *b1, *bcat, *S, *gamma, *beta;  // b1 [F], bo + b2 [D], DCN branch S fp32 [BT, D], LN affine [D]
  int M, D, F, num_sms;
  bool pdl;
};
cudaError_t launch_ens_ffn_ln(const EnsFfnArgs& a, cudaStream_t s);

// ---- K7: multi-head self-attention over the 64 tokens of each example (config 4) ------------------
// qkv [B*S, 3*D] bf16 (Q | K | V, head h at columns h*64 of each), out [B*S, D] bf16; S = 64, dh = 64.
cudaError_t launch_mha64(const __nv_bfloat16* qkv, __nv_bfloat16* out, int out_ld, int B, int n_heads, cudaStream_t s);
// scores[m] = sigmoid(sum_j partial[m][j] + c), j in fixed order (EPI_HEAD_PARTIAL finaliser)
cudaError_t launch_head_finalize(const float* partial, int n_parts, float c, float* scores, int M, cudaStream_t s);

// ---- K5: fused low-rank cross layer (cluster of 4 CTAs per 128-row block, r = 256) ----------------
struct CrossFusedArgs {
  const CUtensorMap* tmXl;   // x_l [M, W] box {64, 128}
  const CUtensorMap* tmV;    // V   [r, W] box {64, 256}
  const CUtensorMap* tmT;    // t   [M, r] box {64, 128}
  const CUtensorMap* tmU;    // U   [W, r] box {64, 64}
  const CUtensorMap* tmX0;   // x0  [M, W] box {64, 128}
  const CUtensorMap* tmOut;  // x_{l+1} [M, W] box {64, 32}
  const float* bias;         // b_l fp32 [W]
  float* part;               // fp32 scratch, cross_fused_partial_bytes(max_batch)
  __nv_bfloat16* t_out;      // t [max_batch, r] bf16
  int M, W, R;
  bool pdl;
  unsigned long long* dbg;   // optional per-CTA phase timestamps (CVR_DEBUG_TIMING)
};
size_t cross_fused_partial_bytes(int max_batch);
cudaError_t launch_cross_fused(const CrossFusedArgs& g, cudaStream_t s);

// ---- the whole low-rank cross stack as one persistent dependency-driven kernel ------------------------
struct CrossStackTables {        // device-resident (64-byte aligned), built at cvr_load_weights
  CUtensorMap V[kMaxLayers];     // V_l [r, W], box {64, 64}
  CUtensorMap U[kMaxLayers];     // U_l [W, r], box {64, 64}
  CUtensorMap xa, xb;            // layer outputs (A operand / x_l epilogue input), box {64, 128}
  CUtensorMap t;                 // t [max_batch, r], box {64, 128}
};
struct CrossStackArgs {
  __nv_bfloat16* xa;
  __nv_bfloat16* xb;
  __nv_bfloat16* t;
  const float* bias[kMaxLayers];
  int* done;                     // [2L][ceil(M/128)] completion counters (zeroed per launch)
  int M, W, R, L, num_sms;
  unsigned long long* dbg;       // optional [grid][32] timestamps (CVR_DEBUG_TIMING)
};
cudaError_t launch_cross_stack(const CUtensorMap* tmX0, const CrossStackTables* d_tables, const CrossStackArgs& a,
                               cudaStream_t s);

// host: encode a 2-D bf16 K-major tensor map [rows, cols] (row stride ld elements) with box
// {64, box_rows} and 128-byte swizzle.
// fp32 [rows, cols] (row stride ld elements), box {32 columns, 32 rows}, 128-byte swizzle: the staged fp32 epilogue
// stores (EPI_CROSS_F32)
int encode_tmap_f32_store(CUtensorMap* tm, const void* ptr, int64_t rows, int64_t cols, int64_t ld, const char** err);
int encode_tmap_bf16(CUtensorMap* tm, const void* ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows,
                     const char** err);

}  // namespace cvr
