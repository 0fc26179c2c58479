/*
 * cvr.h -- C ABI of libcvr.so, the B200 (sm_100a) scoring hot path of the scaled
 * search-CVR model of arxiv/paper_2605_29232 (PAPER.md = the paper's LaTeX source).
 *
 * The path for one batch of B candidate items:
 *   S2 embedding-bag gather + sum-pool   p[b,t,:] = sum_{j in bag(t,b)} E_t[idx_j,:]
 *        PAPER.md:96 (§2.1 "Each categorical feature is designated to an embedding layer");
 *        BASELINE.json north star (a) "multi-hot embedding-bag gather and sum-pool".
 *   S3 dense normalisation + concat      x0 = [p_0 | ... | p_{T-1} | (x - mu)/sigma]
 *        PAPER.md:95 ("normal standardization"), PAPER.md:227 (x_0).
 *   S4 pooled all-to-all (sharded tables only)  -- BASELINE.json configs[2].
 *   S5 DCN-v2 cross layers               x_{l+1} = x0 * (W_l x_l + b_l) + x_l       (full rank)
 *                                        x_{l+1} = x0 * (U_l (V_l x_l) + b_l) + x_l (low rank)
 *        PAPER.md:116-119 (eq:dcnv2) and PAPER.md:225 (§3.1 "The Deep and Cross Family").
 *   S6 MLP tower                         h_{i+1} = ReLU(M_i h_i + c_i)   PAPER.md:229-233.
 *   S7 head                              score = sigmoid(m . h + c)      BASELINE.json north star.
 *   S9 decoupled execution: the embedding stage of batch k+1 overlaps the dense stage of
 *      batch k (§4.5 "Hybrid CPU-GPU Execution"; BASELINE.json north star).
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 *  - Every function returns an int status (cvr_status) and never throws across the ABI.
 *    cvr_last_error(ctx) returns the per-ctx message of the most recent failure (shape
 *    errors name both the expected and the received shape).
 *  - "d_" pointers are CUDA device pointers, "h_" pointers are host pointers.  The caller
 *    (PyTorch) allocates every device buffer; the library only BORROWS them, except the
 *    workspace contents, which it owns between cvr_set_workspace and cvr_destroy.
 *  - Streams are passed as cvr_stream_t (a cudaStream_t, NULL = legacy default stream).
 *    Calls that take a stream only ENQUEUE work; arguments are validated synchronously
 *    on the host before anything is enqueued (null pointers, batch > max_batch,
 *    nnz > max_nnz, call order -> CVR_E_STATE).
 *  - Bad data that only the device can see (index outside [0, rows_t), offsets not
 *    non-decreasing or outside [0, nnz]) sets a sticky device flag; that bag is written
 *    as zeros, and the NEXT cvr_get_status returns CVR_E_INDEX (error, never a clamp;
 *    SURVEY.md §8(c) A23).
 *  - Input layout:
 *      indices  int32 [nnz]       per-table local row ids (already hashed)
 *      offsets  int32 [T*B + 1]   table-major CSR: bag (t, b) is
 *                                 indices[offsets[t*B+b] .. offsets[t*B+b+1]-1]
 *      dense    fp32  [B, F]      raw log1p'd continuous features (normalised inside)
 *      scores   fp32  [B]         sigmoid outputs
 *      x0       [B, x0_ld]        act dtype, row-major; columns [0, W) hold x0 in the
 *                                 canonical order (tables 0..T-1, then dense 0..F-1),
 *                                 columns [W, x0_ld) are zero padding (x0_ld: cvr_x0_layout).
 *  - One ctx is driven by one host thread; several ctxs may coexist.
 */
#ifndef CVR_H_
#define CVR_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct cvr_ctx cvr_ctx;   /* opaque */
typedef void* cvr_stream_t;       /* a cudaStream_t */

typedef enum {
  CVR_OK = 0,
  CVR_E_ARG = 1,      /* null pointer / out-of-range scalar argument */
  CVR_E_SHAPE = 2,    /* weight or table shape mismatch (message names both shapes) */
  CVR_E_DTYPE = 3,    /* dtype mismatch */
  CVR_E_STATE = 4,    /* call order (e.g. cvr_dense before weights are loaded) */
  CVR_E_INDEX = 5,    /* device saw an out-of-range index or malformed offsets */
  CVR_E_NOMEM = 6,    /* workspace too small */
  CVR_E_CUDA = 7,     /* CUDA runtime / driver failure (message has the CUDA text) */
  CVR_E_NCCL = 8,     /* NCCL failure */
  CVR_E_OVERLOAD = 9, /* serving queue full (batcher) */
  CVR_E_UNSUPPORTED = 10 /* model shape outside what the kernels support */
} cvr_status;

typedef enum { CVR_F32 = 0, CVR_BF16 = 1, CVR_F16 = 2 } cvr_dtype;

/* An NCCL unique id (ncclUniqueId: 128 opaque bytes), created by one rank (cvr_comm_unique_id) and handed to every
 * rank by the caller's process group. */
typedef struct { char internal[128]; } cvr_nccl_id;

#define CVR_EXECUTOR_SLOTS 2  /* x0 slots (and per-call blocks, host-fed staging) of cvr_score / cvr_score_host */

typedef enum {
  CVR_DCN_FULL = 0,     /* full-rank cross with bias, fp32 SIMT path (config 1)      */
  CVR_DCN_LOWRANK = 1,  /* low-rank cross, bf16 tcgen05 path (configs 2, 3, 5)       */
  CVR_ENSEMBLE = 2,     /* DCN || MHA || FFN, summed + layer-normed (config 4)       */
  CVR_MASKNET = 3       /* ReLU input projection + instance-guided mask blocks, bf16 tcgen05 path:
                         *   x0' = ReLU(W_in x0 + b_in)
                         *   x_{s+1} = (U ReLU(V x0' + c) + b) * x_s     PAPER.md:226 (no residual, :363)
                         * n_parallel branches of n_cross blocks each (x_0 = x0'), outputs concatenated
                         * (PAPER.md:229-233), then the MLP tower + head     */
} cvr_backbone;

/* Model + run description; copied by cvr_create (the arrays need not outlive the call). */
typedef struct {
  int n_tables;             /* T (all tables of the model, also in sharded mode)        */
  const int64_t* rows;      /* [T] rows per table                                       */
  int dim;                  /* d, embedding dim (same for every table)                  */
  int emb_dtype;            /* cvr_dtype of the table rows                              */
  int n_dense;              /* F continuous features                                    */
  int act_dtype;            /* CVR_F32 (DCN_FULL) or CVR_BF16                            */
  int backbone;             /* cvr_backbone                                             */
  int n_cross;              /* number of cross (or ensemble) layers                     */
  int cross_rank;           /* r for DCN_LOWRANK / ENSEMBLE, 0 for DCN_FULL             */
  int n_mlp;                /* hidden layers of the MLP tower                           */
  const int* mlp_dims;      /* [n_mlp] hidden widths; the width-1 head is implicit      */
  int n_heads;              /* ENSEMBLE only                                            */
  int ffn_dim;              /* ENSEMBLE only                                            */
  int max_batch;            /* largest B any call will pass                             */
  int64_t max_nnz;          /* largest nnz any call will pass (host-fed staging)        */
  int world_size;           /* 1 = unsharded; >1 = table-wise sharding (t -> t % N)     */
  int rank;                 /* this process's rank when world_size > 1                  */
  int cross_width;          /* MASKNET: projected cross width W' (multiple of 64); else 0 */
  int n_parallel;           /* MASKNET: parallel branches P (n_cross = blocks per branch); else 0 */
} cvr_model_desc;

/* -- lifecycle ------------------------------------------------------------------------ */
int cvr_create(const cvr_model_desc* desc, cvr_ctx** out);
int cvr_destroy(cvr_ctx* ctx);
const char* cvr_last_error(const cvr_ctx* ctx);
const char* cvr_status_string(int status);
/* Library version string and the compiled device architecture ("sm_100a"). */
const char* cvr_version(void);

/* Device workspace (weights, x0 slots, intermediates, staging, flags); caller-allocated,
 * >= 256-byte aligned.  Must be set before cvr_load_weights.  With option "lanes" L > 1 (set before this call) the
 * size covers every lane (each lane holds its own copy of everything but the borrowed tables). */
int cvr_workspace_bytes(const cvr_ctx* ctx, size_t* bytes);
int cvr_set_workspace(cvr_ctx* ctx, void* d_ws, size_t bytes);

/* x0 row stride (elements) and dtype used by cvr_embed / cvr_dense. */
int cvr_x0_layout(const cvr_ctx* ctx, int* x0_ld, int* x0_dtype);

/* -- parameters ----------------------------------------------------------------------- */
/* Borrow n embedding tables: table_ids[i] in [0, T) (in sharded mode only the tables this
 * rank owns, t % world_size == rank); d_rows[i] is [rows_t, d] of emb_dtype with a row
 * stride of row_stride_bytes[i] (multiple of 16, base 16-byte aligned).  The pointers must
 * outlive the ctx.  Sharded mode requires exactly the owned tables. */
int cvr_load_tables(cvr_ctx* ctx, int n, const int* table_ids, const void* const* d_rows,
                    const int64_t* row_stride_bytes);

/* COPY n named parameters into the workspace (repacked as the kernels need).  Names and
 * [out, in] shapes:
 *   "norm/mean" [F], "norm/std" [F]                                   (fp32)
 *   DCN_FULL:    "dcn/<l>/W" [W, W], "dcn/<l>/b" [W]
 *   DCN_LOWRANK: "dcn/<l>/V" [r, W], "dcn/<l>/U" [W, r], "dcn/<l>/b" [W]
 *   ENSEMBLE:    "ens/<l>/dcn/{V,U,b}", "ens/<l>/mha/{Wqkv,bqkv,Wo,bo}",
 *                "ens/<l>/ffn/{W1,b1,W2,b2}", "ens/<l>/ln/{gamma,beta}"
 *   MASKNET:     "proj/W" [W', W], "proj/b" [W'], for branch p < P and block q < n_cross:
 *                "mask/<p>/<q>/V" [r, W'], ".../c" [r], ".../U" [W', r], ".../b" [W'];
 *                the MLP input width is P * W'
 *   "mlp/<i>/W" [h_i, h_{i-1}], "mlp/<i>/b" [h_i], "head/w" [1, h_last], "head/b" [1]
 * shapes is flattened: entry i has ndims[i] extents starting at the running offset.
 * Every expected name must be present exactly once (else CVR_E_SHAPE); dtypes must be
 * act_dtype (the norm/ entries fp32).  Synchronous; the caller may free its tensors afterwards. */
int cvr_load_weights(cvr_ctx* ctx, int n, const char* const* names, const void* const* d_ptrs,
                     const int* dtypes, const int* ndims, const int64_t* shapes);

/* -- the hot path ---------------------------------------------------------------------- */
/* S2+S3: pooled embeddings + normalised dense features into d_x0 [batch, x0_ld].
 * Unsharded only (sharded: cvr_embed_shard + cvr_exchange). */
int cvr_embed(cvr_ctx* ctx, const int32_t* d_indices, const int32_t* d_offsets, int64_t nnz,
              int batch, const float* d_dense, void* d_x0, cvr_stream_t stream);

/* S5-S7 on d_x0 [batch, x0_ld] -> d_scores [batch] fp32. */
int cvr_dense(cvr_ctx* ctx, const void* d_x0, int batch, float* d_scores, cvr_stream_t stream);

/* S2-S7 for one batch using the ctx's CVR_EXECUTOR_SLOTS x0 slots (batch k uses slot k % CVR_EXECUTOR_SLOTS): the
 * embed stage runs on s_embed, the dense stage on s_dense, with event edges embed(k) -> dense(k) and
 * dense(k) -> embed(k + CVR_EXECUTOR_SLOTS) (slot reuse).  Back-to-back calls therefore overlap the embed stage of
 * batch k+1 with the dense stage of batch k (S9; "Hybrid CPU-GPU
 * Execution").
 * Each stage is one CUDA graph per (x0 slot, grid-size bucket), captured at its first use and replayed for every
 * later batch: the batch's pointers and row count are written to a per-slot argument block in the workspace (a
 * one-thread kernel on s_embed) that every kernel of both stages reads, so no pointer or size is baked into a graph;
 * the bucket (batch rounded up to a power of two >= 128, capped at max_batch) only sizes the grids (option
 * "graphs" [1]).  The pointers must stay valid until s_dense has passed this batch.
 * Executor lanes (option "lanes" = L > 1): consecutive calls are dealt round-robin to L independent pipelines of
 * the model (each with its own slots, intermediates and graphs, on its own pair of library streams created with
 * the priorities of s_embed / s_dense): the call's work starts after everything enqueued on s_embed so far (the
 * inputs AND d_scores must be ready there) and s_dense waits for its end, so the dense stages of consecutive
 * batches may run concurrently (throughput up, per-batch latency up). */
int cvr_score(cvr_ctx* ctx, const int32_t* d_indices, const int32_t* d_offsets, int64_t nnz,
              int batch, const float* d_dense, float* d_scores, cvr_stream_t s_embed,
              cvr_stream_t s_dense);

/* Capture (without running anything) the executor graphs of every grid-size bucket up to max_rows, for both x0
 * slots and both stages (and the keys-mode embed stage when every table has a hash vocab), so that no batch of a
 * serving run pays a capture; the graphs read their batch from the call block at replay time.  Streams are only
 * used to capture on (non-NULL).  CVR_E_ARG if max_rows is outside [1, max_batch]. */
int cvr_warm_graphs(cvr_ctx* ctx, int max_rows, cvr_stream_t s_embed, cvr_stream_t s_dense);

/* Host-fed variant (S1 + S2-S7 + S8): h_* are host buffers (pinned for async copies);
 * the H2D copies of this batch run on s_copy into double-buffered device staging,
 * then as cvr_score.  S8: when h_scores is page-locked (mapped) memory the head kernel stores
 * the scores straight into it over PCIe (zero-copy; option "zero_copy_scores" [1]), otherwise
 * they are copied D2H on s_dense.  Returns after enqueueing; h_scores is valid once s_dense
 * has been synchronised.  The batch's pinned h_scores must not be reused by another call in
 * flight (one scores buffer per batch in flight, as for the inputs). */
int cvr_score_host(cvr_ctx* ctx, const int32_t* h_indices, const int32_t* h_offsets, int64_t nnz,
                   int batch, const float* h_dense, float* h_scores, cvr_stream_t s_copy,
                   cvr_stream_t s_embed, cvr_stream_t s_dense);

/* Synchronise `stream`, read and clear the sticky device flag: CVR_E_INDEX if any kernel
 * since the last call saw bad indices/offsets, CVR_E_CUDA on an asynchronous CUDA error. */
int cvr_get_status(cvr_ctx* ctx, cvr_stream_t stream);

/* -- table-wise sharding (world_size > 1; BASELINE.json configs[2]) ---------------------- */
/* Bytes of the send and receive buffers for a global batch (per rank). */
int cvr_shard_buffer_bytes(const cvr_ctx* ctx, int batch_global, size_t* send_bytes, size_t* recv_bytes);

/* S2 for the local tables over the GLOBAL batch, written destination-major into d_send:
 * [dst][b_local][t_local][d] (act dtype, t_local padded to max tables per rank), plus
 * S3 for this rank's batch slice [rank*B/N, (rank+1)*B/N) into d_x0 (dense columns).
 * indices/offsets cover the local tables (offsets [T_local*B_global + 1]); d_dense is the
 * local slice [B/N, F]. */
int cvr_embed_shard(cvr_ctx* ctx, const int32_t* d_indices, const int32_t* d_offsets, int64_t nnz,
                    int batch_global, const float* d_dense, void* d_send, void* d_x0,
                    cvr_stream_t stream);

/* -- fused exchange (V3 of SURVEY.md §8(e), §8(f) #4): no send / receive buffers, no all-to-all ----------
 * Each rank owns TWO x0 slots ([batch_global / N, x0_ld] each, the buffers it passes to cvr_dense; batch epoch e
 * uses slot e % 2) and two uint32 [N] flag arrays, zero-initialised once: ready[src] and free[dst].
 * cvr_set_peers: d_peer_x0[slot * N + dst] is rank dst's x0 slot mapped into this process (cvr_ipc_open_handle
 * of its cvr_ipc_get_handle; this rank's own buffers for dst == rank), d_peer_ready[dst] / d_peer_free[dst]
 * rank dst's flag arrays, d_local_ready / d_local_free this rank's.  n == world_size > 1.
 * cvr_embed_fused (epoch e = 1, 2, ...): waits until free[dst] >= e - 2 for every dst (each owner has finished
 * the dense stage that read slot e % 2 two batches ago), then the gather kernel writes each pooled bag (local
 * table t, global example b) straight into d_peer_x0[(e % 2) * N + b / (B/N)] at row b % (B/N), columns
 * (t*N + rank)*d (the canonical x0 layout; round-robin placement, A18) and the normalised dense features of this
 * rank's slice into d_x0 (this rank's slot e % 2), then stores ready[rank] = e on every rank (release, system
 * scope, after a system fence).
 * cvr_wait_peers(e): enqueues a wait until this rank's ready[src] >= e for every src (acquire, system scope);
 * after it the slot holds the complete canonical x0 slice and cvr_dense may run on it.
 * cvr_release_peers(e): after that dense stage, stores free[rank] = e on every rank.
 * Pooled values are bit-identical to cvr_embed / the NCCL path (same per-bag order; the exchange is a store). */
int cvr_set_peers(cvr_ctx* ctx, int n, void* const* d_peer_x0, uint32_t* const* d_peer_ready,
                  uint32_t* const* d_peer_free, uint32_t* d_local_ready, uint32_t* d_local_free);
int cvr_embed_fused(cvr_ctx* ctx, const int32_t* d_indices, const int32_t* d_offsets, int64_t nnz, int batch_global,
                    const float* d_dense, void* d_x0, uint32_t epoch, cvr_stream_t stream);
int cvr_wait_peers(cvr_ctx* ctx, uint32_t epoch, cvr_stream_t stream);
int cvr_release_peers(cvr_ctx* ctx, uint32_t epoch, cvr_stream_t stream);
/* CUDA IPC for the peer mappings.  cvr_ipc_get_handle writes CVR_IPC_HANDLE_BYTES: the 64-byte CUDA IPC handle of
 * the allocation that CONTAINS d_ptr plus the 8-byte offset of d_ptr inside it (a caching allocator may sub-allocate
 * tensors); cvr_ipc_open_handle maps the allocation in another process of the node (peer access enabled lazily) and
 * returns the mapped base + offset; cvr_ipc_close_handle(that pointer) unmaps it once no opened pointer of the same
 * allocation remains.  CVR_E_CUDA on a CUDA failure, CVR_E_ARG on an unknown pointer. */
#define CVR_IPC_HANDLE_BYTES 72
int cvr_ipc_get_handle(const void* d_ptr, void* handle);
int cvr_ipc_open_handle(const void* handle, void** d_ptr);
int cvr_ipc_close_handle(void* d_ptr);

/* -- S4 pooled all-to-all over the library's own NCCL communicator (BASELINE.json
 * configs[2] "pooled embeddings exchanged by all-to-all") ----------------------------------------------------------
 * NCCL is resolved at run time (the process's libnccl.so.2 -- PyTorch's -- or CVR_NCCL_LIB); CVR_E_NCCL if absent.
 * cvr_comm_unique_id: a new unique id (call on one rank, broadcast it).  cvr_comm_init: ncclCommInitRank for this
 * ctx (collective over the world_size ranks; world / rank must equal the ctx's; the current CUDA device is used).
 * cvr_exchange: one grouped ncclSend / ncclRecv per peer on `stream`: chunk dst of d_send ([dst][b_local][t_slot][d],
 * as written by cvr_embed_shard, cvr_shard_buffer_bytes each) goes to rank dst, chunk src of d_recv comes from rank
 * src; then the unpack kernel writes the received pooled rows into the canonical x0 columns of d_x0_local (this
 * rank's slice [batch_global / N, x0_ld], whose dense columns cvr_embed_shard already wrote).  The payload is the
 * pooled rows verbatim (P11: bit-identical to the unsharded path).  CVR_E_STATE before cvr_comm_init. */
int cvr_comm_unique_id(cvr_nccl_id* id);
int cvr_comm_init(cvr_ctx* ctx, const cvr_nccl_id* id, int world, int rank);
int cvr_exchange(cvr_ctx* ctx, const void* d_send, void* d_recv, int batch_global, void* d_x0_local,
                 cvr_stream_t stream);

/* Unpack received source-major chunks d_recv [src][b_local][t_slot][d] into the canonical
 * x0 columns of the local slice (V1 of SURVEY.md §8(e)); cvr_exchange runs it after its all-to-all. */
int cvr_unpack_shard(cvr_ctx* ctx, const void* d_recv, int batch_global, void* d_x0, cvr_stream_t stream);

/* Options (defaults in brackets): "graphs" [1] replay the executor stages of cvr_score / cvr_score_host as
 * CUDA graphs (see cvr_score); "pdl" [1] launch dependent GEMMs with programmatic stream serialization;
 * "prefetch_b" [1] each GEMM issues its first ring stages' weight loads before waiting for the previous kernel;
 * "embed_bps" [0 = uncapped] embedding CTAs per SM inside the executor; "xv_bn" [0 = by wave count] N tile of
 * t = x_l V^T (64, 128, 256); "u_bn" [192] N tile of the low-rank U GEMM (192 when W % 192 == 0, else 64);
 * "epw" [0 for DCN_LOWRANK, else 2] epilogue warps per TMEM quadrant: 0 one, 1 up to 4 (one 64-column sub-tile
 * each), 2 split only when a CTA runs <= 2 tiles; "zero_copy_scores" [1] cvr_score_host stores the scores straight into page-locked h_scores;
 * config 4: "pair" [1] 2-CTA (cta_group::2) tiles, "ens_u_bn" [128] N tile of the DCN U GEMM, "ens_fused_attn" [1]
 * the QKV projection + attention as one GEMM (else QKV GEMM + mha64), "ens_attn_tc" [1] that GEMM's attention on
 * tcgen05 (S = Q K^T, O = P V as UMMAs in TMEM; else mma.sync in the epilogue), "f32_tma_store" [1] the fp32 DCN-branch
 * output through staged TMA stores, "ens_xv_wave" [1] t = X V^T as one wave of 128 x 256 tiles, "ens_ffn_fused" [0]
 * FFN1 + out-projection + FFN2 + LN as one kernel (hidden activations never stored; measured slower); MaskNet:
 * "mask_grouped" [1] parallel blocks as one grouped GEMM.  Every variant is bit-identical to the default.
 * "lanes" [1] executor lanes (1-4, see cvr_score): only before cvr_set_workspace (else CVR_E_STATE), unsharded
 * only; sub-contexts are created here and every later option, table, weight and feature-spec call is applied to
 * all lanes.  Unknown key or bad value -> CVR_E_ARG. */
int cvr_set_option(cvr_ctx* ctx, const char* key, int64_t value);

/* -- utility ----------------------------------------------------------------------------------
 * C[M, N] = A[M, K] . B[N, K]^T on the same tcgen05/TMA kernel the dense stage uses (tests and
 * tile tuning): bf16 row-major operands with leading dimensions lda/ldb/ldc (elements, multiples
 * of 8), fp32 accumulation, bf16 output; epi 0 = plain store, 1 = ReLU(C + bias[N]) (fp32 bias, 16-byte
 * aligned, else CVR_E_ARG).
 * K % 64 == 0, N % bn == 0, bn in {64, 128, 256}; epi | 0x100 selects the 2-CTA (cta_group::2, 256-row
 * tile per CTA pair) variant.  Enqueued on `stream`. */
int cvr_gemm_bf16(const void* d_A, int64_t lda, const void* d_B, int64_t ldb, void* d_C, int64_t ldc, int M, int N,
                  int K, int epi, const float* d_bias, int bn, cvr_stream_t stream);

/* -- serving: stage 0 batch assembly (host) -------------------------------
 * Concatenate n_req requests (request r = n_items[r] candidate items of one query, PAPER.md:1560
 * "Client-Side Batching") into one batch in the library's input layout.  Request r carries its own
 * table-major CSR (h_offsets[r] [T*n_r + 1], h_indices[r]) and dense rows h_dense[r] [n_r, F]
 * (host memory).  Output: out_offsets [T*B + 1], out_indices (capacity out_indices_cap), out_dense
 * [B, F] with B = sum n_items, items in request order (the scatter map is implicit: request r owns
 * rows [sum_{q<r} n_q, sum_{q<=r} n_q)).  Pure host memcpy work (typically into pinned staging);
 * out_offsets / out_dense have room for out_batch_cap items; CVR_E_NOMEM if B > out_batch_cap or the indices do not
 * fit, CVR_E_INDEX if a request's offsets are negative or decrease. */
int cvr_concat_requests(int n_req, int n_tables, int n_dense, const int* n_items, const int32_t* const* h_offsets,
                        const int32_t* const* h_indices, const float* const* h_dense, int out_batch_cap,
                        int32_t* out_offsets, int32_t* out_indices, int64_t out_indices_cap, float* out_dense,
                        int64_t* out_nnz);

/* Gather n items of a host-resident item pool (table-major CSR pool_offsets [T*P + 1],
 * pool_indices, pool_dense [P, F]; a feature store) into one batch in the library's input layout:
 * out_offsets [T*n + 1], out_indices, out_dense [n, F], item i of the batch = pool item item_ids[i].
 * out_offsets / out_dense have room for out_batch_cap items.  Host-only; CVR_E_INDEX on an item id outside
 * [0, P), CVR_E_NOMEM if n > out_batch_cap or the indices do not fit. */
int cvr_gather_items(int n_tables, int n_dense, int64_t pool_size, const int32_t* pool_offsets,
                     const int32_t* pool_indices, const float* pool_dense, int n, const int32_t* item_ids,
                     int out_batch_cap, int32_t* out_offsets, int32_t* out_indices, int64_t out_indices_cap,
                     float* out_dense, int64_t* out_nnz);

/* -- serving: the native dynamic-batching loop (SURVEY.md §8(a) S0 + S9; "Server-Side Batching",
 * Table 6) ------------------------------------------------------------------
 * Batcher rule (identical to serving.DynamicBatcher): requests are never split; a request with more than max_items
 * items or arriving at a full queue (queue_capacity requests) is rejected (latency +inf); a batch is
 * dispatched when the queued items reach max_items or the OLDEST queued request has waited window_s, and holds the
 * longest FIFO prefix of whole requests with sum(items) <= max_items (and <= max_requests requests when > 0;
 * max_requests = 1 with window_s = 0 is Table 6's "w/o dynamic batching" row). */
typedef struct {
  double window_s;        /* coalescing window, anchored at the oldest queued request                         */
  int max_items;          /* batch cap (<= the ctx's max_batch)                                               */
  int max_requests;       /* 0 = no limit                                                                     */
  int queue_capacity;     /* queued requests before overload rejection                                       */
  int host_slots;         /* batches in flight (pinned staging slots), 1..16                                  */
  int64_t max_nnz;        /* index capacity of a slot (<= the ctx's max_nnz)                                  */
  double abort_after_s;   /* > 0: stop once the oldest queued request has waited this long (overload probe)    */
} cvr_serve_config;

typedef struct {
  int64_t rejected;       /* requests rejected at admission                                                   */
  int aborted;            /* 1 if abort_after_s stopped the run (unserved requests keep latency +inf)          */
  int64_t items_served;
  double host_dispatch_s; /* host time spent assembling + enqueueing batches                                  */
  double wall_s;          /* from the trace's time origin to the last completion                              */
  double max_dispatch_s;  /* the longest single batch assembly + enqueue                                     */
  double max_gather_s;    /* the longest single batch assembly (cvr_gather_items)                             */
  int64_t loop_gaps_1ms;  /* polling-loop iterations that took > 1 ms (the host thread was held up)           */
} cvr_serve_stats;

/* Serve an open-loop trace on ONE host thread: request r arrives at t_arrival[r] seconds (non-decreasing; the
 * origin is 10 ms after the call starts) with n_items[r] candidate items, pool item ids
 * item_ids[item_start[r] .. item_start[r] + n_items[r]) of the host item pool (table-major CSR pool_offsets
 * [T*P + 1], pool_indices, pool_dense [P, F], as cvr_gather_items).  Each dispatched batch is assembled into one of
 * host_slots page-locked staging slots (cvr_gather_items) and enqueued with cvr_score_host on the three streams
 * (the scores are stored straight into the slot's mapped buffer); a CUDA event per slot marks completion, polled
 * without blocking.  Outputs: latency[r] = completion seen on the host - t_arrival[r] (s; +inf if rejected or not
 * served), scores_out (optional, [sum n_items]) at item_start[r], batch_sizes[b] (capacity n_req) and *n_batches,
 * stats.  Synchronous (returns when every batch has completed). */
int cvr_serve_trace(cvr_ctx* ctx, const cvr_serve_config* cfg, int n_tables, int n_dense, int64_t pool_size,
                    const int32_t* pool_offsets, const int32_t* pool_indices, const float* pool_dense, int n_req,
                    const double* t_arrival, const int32_t* n_items, const int64_t* item_start,
                    const int32_t* item_ids, double* latency, float* scores_out, int32_t* batch_sizes,
                    int* n_batches, cvr_serve_stats* stats, cvr_stream_t s_copy, cvr_stream_t s_embed,
                    cvr_stream_t s_dense);

/* The same batcher on a simulated clock: one server whose batch of n items takes
 * service_fixed_s + service_per_item_s * n seconds; a batch is dispatched when the batcher releases it and the
 * server is free.  latency[r] (+inf if rejected), batch_of[r] (-1 if rejected), dispatch_time[b] (capacity n_req),
 * *n_batches.  Host only (tests). */
int cvr_batcher_simulate(int n_req, const double* t_arrival, const int32_t* n_items, double window_s, int max_items,
                         int max_requests, int queue_capacity, double service_fixed_s, double service_per_item_s,
                         double* latency, int32_t* batch_of, double* dispatch_time, int* n_batches);

/* -- feature front end -----------------------------------------------------
 * Per model table t (n == T): vocab[t] > 0 puts the table in keys mode -- cvr_embed_keys hashes each raw
 * 64-bit key on the device, row = FNV-1a 64 over the key's 8 big-endian bytes mod vocab[t] (
 * PAPER.md:271 "hashing trick"), the MISSING key 0xFFFFFFFFFFFFFFFF maps to the `unseen' row vocab[t]
 * (PAPER.md:287), so rows[t] >= vocab[t] + 1 is required (else CVR_E_SHAPE); vocab[t] = 0 keeps
 * row ids.  pool_mode[t] = 1 mean-pools the bag (sum / length, fp32; "average pooling"), 0 sums;
 * empty bags pool to 0 either way; mean also applies to cvr_embed / cvr_score.  Host call, synchronous. */
int cvr_set_feature_spec(cvr_ctx* ctx, int n, const int64_t* vocab, const int* pool_mode);

/* S2+S3 in keys mode: d_keys uint64 [nnz] raw keys in the table-major CSR of d_offsets (as cvr_embed's
 * indices); every table must be in keys mode (CVR_E_STATE otherwise).  Otherwise as cvr_embed. */
int cvr_embed_keys(cvr_ctx* ctx, const uint64_t* d_keys, const int32_t* d_offsets, int64_t nnz, int batch,
                   const float* d_dense, void* d_x0, cvr_stream_t stream);

/* cvr_score in keys mode: the embedding stage hashes d_keys (as cvr_embed_keys); same executor, streams
 * and ordering as cvr_score. */
int cvr_score_keys(cvr_ctx* ctx, const uint64_t* d_keys, const int32_t* d_offsets, int64_t nnz, int batch,
                   const float* d_dense, float* d_scores, cvr_stream_t s_embed, cvr_stream_t s_dense);

/* Host batch assembly for text features ("tokenized into character n-grams"): the overlapping
 * n-byte grams (1 <= n <= 8) of each of n_texts byte strings, each packed big-endian into a 64-bit key, into
 * out_keys (capacity out_cap) with CSR out_offsets [n_texts + 1]; a string shorter than n gives an empty bag.
 * CVR_E_NOMEM if out_cap is too small. */
int cvr_text_ngram_keys(int n_texts, const char* const* texts, const int32_t* lens, int n, uint64_t* out_keys,
                        int64_t out_cap, int32_t* out_offsets, int64_t* out_nnz);

/* Host batch assembly for sequential features: keep the most recent max_len keys of each bag
 * (bags list oldest first); out_keys needs room for min(len, max_len) per bag.  CVR_E_INDEX on decreasing
 * offsets. */
int cvr_truncate_bags(int n_bags, const int32_t* offsets, const uint64_t* keys, int max_len, int32_t* out_offsets,
                      uint64_t* out_keys, int64_t* out_nnz);

/* -- accounting / measurement -------------------------------------------------------------- */
/* Number of kernels this ctx has launched since creation (every entry point counts its launches). */
int cvr_launch_count(const cvr_ctx* ctx, int64_t* n);

typedef struct {
  char name[32];     /* kernel role: embed_bag_pool, gemm_xV, gemm_tU_cross, gemm_mlp_relu, ... */
  int64_t launches;
  double total_ms;   /* sum of CUDA-event durations measured on the launching stream */
  double min_ms, max_ms;
} cvr_kernel_stat;

/* What the executor's kernels consumed: the per-call argument block of x0 slot `slot` (batch k used slot
 * k % CVR_EXECUTOR_SLOTS; with L lanes slot is in [0, L * CVR_EXECUTOR_SLOTS): call n ran on lane n % L, in that
 * lane's slot (n / L) % CVR_EXECUTOR_SLOTS, flat index lane * CVR_EXECUTOR_SLOTS + slot) as
 * the device holds it -- the device pointers and sizes the embed / dense graphs read (P12: the caller hashes the
 * arrays behind them) -- and how many executor graphs this ctx has captured (all lanes).  Synchronous. */
typedef struct {
  const int32_t* d_indices;
  const uint64_t* d_keys;
  const int32_t* d_offsets;
  const float* d_dense;
  float* d_scores;
  int64_t nnz;
  int batch;
  int64_t graph_captures;
} cvr_call_record;
int cvr_call_info(const cvr_ctx* ctx, int slot, cvr_call_record* out);

/* Measurement: run the dense stage on d_x0 [batch, x0_ld] launching ONLY the tcgen05 GEMMs of kernel role `role`
 * (a cvr_kernel_stat name, e.g. "gemm_tU_cross"), each of them `reps` times back to back on `stream` with the stage's
 * programmatic (PDL) launches -- the GEMMs are idempotent given the buffers a full stage left behind (call cvr_dense
 * on the same x0 first), so CUDA events around the call give the role's steady-state per-launch time inside a
 * PDL chain without event pairs between kernels.  *n_launched = launches enqueued.  CVR_E_UNSUPPORTED on the fp32
 * path. */
int cvr_repeat_kernel(cvr_ctx* ctx, const char* role, int reps, const void* d_x0, int batch, cvr_stream_t stream,
                      int* n_launched);

/* Record a CUDA event pair around each of the next max_launches kernel launches (on the stream
 * the kernel is launched on).  cvr_profile_end synchronises on those events, aggregates them per
 * kernel role into out[0 .. min(*n_out, max_out)) and stops recording. */
int cvr_profile_begin(cvr_ctx* ctx, int max_launches);
int cvr_profile_end(cvr_ctx* ctx, cvr_kernel_stat* out, int max_out, int* n_out);

#ifdef __cplusplus
}
#endif
#endif /* CVR_H_ */
