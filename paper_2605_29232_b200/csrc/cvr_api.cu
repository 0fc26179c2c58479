// cvr_api.cu -- the C ABI of libcvr.so (include/cvr.h): context, argument validation, workspace
// carving, weight repacking, the dense-stage schedule and the decoupled two-stream executor
// ("Hybrid CPU-GPU Execution" / BASELINE.json north star
// "embedding lookups for batch k+1 overlap the dense stage of batch k").
//
// No CUDA call is made before cvr_set_workspace, so creation / validation / layout queries work
// on a host without a GPU.
#include <cudaTypedefs.h>
#include <omp.h>
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/cvr.h"
#include "cvr_kernels.cuh"

using namespace cvr;

enum KernelId {
  K_EMBED = 0, K_GEMM_V, K_GEMM_U, K_GEMM_MLP, K_GEMM_HEAD, K_DENSE_F32, K_UNPACK, K_ENS_QKV, K_MHA,
  K_ENS_FFN1, K_ENS_FFN2_LN, K_HEAD_FIN, K_MASK_PROJ, K_MASK_HIDDEN, K_MASK_MUL, K_ENS_QKV_ATTN, K_SET_CALL,
  K_PEER, K_ENS_FFN_FUSED, K_COUNT
};
static const char* kKernelNames[K_COUNT] = {
    "embed_bag_pool", "gemm_xV",  "gemm_tU_cross",  "gemm_mlp_relu", "gemm_mlp_head", "dense_f32_dcn",
    "shard_unpack",   "gemm_ens_qkv", "mha64", "gemm_ens_ffn1", "gemm_ens_ffn2_ln", "head_finalize",
    "gemm_mask_proj", "gemm_mask_hidden", "gemm_mask_mul", "gemm_ens_qkv_attn", "set_call", "peer_flags",
    "gemm_ens_ffn_fused"};

namespace {

size_t elt_size(int dt) { return dt == CVR_F32 ? 4 : 2; }
int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

struct WSlot {
  std::string name;
  std::vector<int64_t> shape;  // expected [out, in] as passed by the caller
  int dtype;                   // expected caller dtype
  size_t off = 0;              // offset of the repacked copy in the workspace
  size_t bytes = 0;
  bool loaded = false;
};

struct GemmPlan {
  int N, K, BN;
  Epi epi;
  bool pair = false;  // 2-CTA (cta_group::2) tiles; B map box = BN/2 rows
  CUtensorMap tmB;
};

// NCCL, resolved at run time (dlopen of the libnccl.so.2 the process already has -- PyTorch's -- or the system
// one): no link-time dependency, so the library still loads and validates on a host without NCCL / a GPU.
struct Nccl {
  void* dl = nullptr;
  int (*getUniqueId)(void*) = nullptr;
  int (*commInitRank)(void**, int, cvr_nccl_id, int) = nullptr;
  int (*commDestroy)(void*) = nullptr;
  int (*groupStart)() = nullptr;
  int (*groupEnd)() = nullptr;
  int (*send)(const void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*recv)(void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  const char* (*errorString)(int) = nullptr;
  std::string why;
  bool load() {
    if (dl) return true;
    const char* env = getenv("CVR_NCCL_LIB");
    const char* names[] = {env, "libnccl.so.2", "libnccl.so"};
    for (const char* n : names) {
      if (!n) continue;
      dl = dlopen(n, RTLD_NOW | RTLD_NOLOAD);  // the copy already in the process (torch's) first
      if (!dl) dl = dlopen(n, RTLD_NOW | RTLD_LOCAL);
      if (dl) break;
    }
    if (!dl) {
      why = "libnccl.so.2 not found (set CVR_NCCL_LIB)";
      return false;
    }
    getUniqueId = reinterpret_cast<int (*)(void*)>(dlsym(dl, "ncclGetUniqueId"));
    commInitRank = reinterpret_cast<int (*)(void**, int, cvr_nccl_id, int)>(dlsym(dl, "ncclCommInitRank"));
    commDestroy = reinterpret_cast<int (*)(void*)>(dlsym(dl, "ncclCommDestroy"));
    groupStart = reinterpret_cast<int (*)()>(dlsym(dl, "ncclGroupStart"));
    groupEnd = reinterpret_cast<int (*)()>(dlsym(dl, "ncclGroupEnd"));
    send = reinterpret_cast<int (*)(const void*, size_t, int, int, void*, cudaStream_t)>(dlsym(dl, "ncclSend"));
    recv = reinterpret_cast<int (*)(void*, size_t, int, int, void*, cudaStream_t)>(dlsym(dl, "ncclRecv"));
    errorString = reinterpret_cast<const char* (*)(int)>(dlsym(dl, "ncclGetErrorString"));
    if (!getUniqueId || !commInitRank || !commDestroy || !groupStart || !groupEnd || !send || !recv) {
      why = "libnccl.so.2 lacks ncclSend / ncclRecv / ncclCommInitRank";
      dlclose(dl);
      dl = nullptr;
      return false;
    }
    return true;
  }
  const char* err(int r) { return errorString ? errorString(r) : "nccl error"; }
};
Nccl g_nccl;
constexpr int kNcclUint8 = 1;  // ncclDataType_t ncclUint8 (nccl.h): the exchange moves raw bytes

}  // namespace

struct cvr_ctx {
  // ---- model description
  int T = 0, d = 0, emb_dtype = 0, F = 0, act = 0, backbone = 0, n_cross = 0, r = 0, n_mlp = 0;
  std::vector<int> mlp;
  int n_heads = 0, ffn = 0, max_batch = 0;
  int64_t max_nnz = 0;
  int world = 1, rank = 0;
  std::vector<int64_t> rows;
  int W = 0;
  int64_t x0_ld = 0;
  // sharding
  std::vector<int> local_tables;
  int T_pad = 0;
  void* nccl_comm = nullptr;        // this ctx's NCCL communicator (cvr_comm_init), the S4 all-to-all
  int comm_world = 0, comm_rank = 0;
  // fused exchange (V3): device table: [2][world] peer x0 slot bases, [world] peer ready-flag arrays, [world] peer
  // free-flag arrays
  size_t off_peers = 0;
  uint32_t* local_ready = nullptr;  // [world]: ready[src] = last epoch whose rows src stored into our x0 slot
  uint32_t* local_free = nullptr;   // [world]: free[dst] = last epoch whose dense stage dst has finished
  bool peers_set = false;
  // ---- state
  std::string err;
  uint8_t* ws = nullptr;
  size_t ws_bytes = 0, ws_need = 0;
  std::vector<WSlot> wslots;
  bool tables_loaded = false, weights_loaded = false;
  std::vector<TableDesc> htables;
  // feature front end (cvr_set_feature_spec): per model table, hash modulus (0 = row ids) and mean pooling
  std::vector<int64_t> tvocab;
  std::vector<int> tmean;
  bool any_mean = false;
  // workspace regions (offsets)
  // executor x0 slots: batch k uses slot k % kSlots.  (Three slots, letting the embed stream run two batches ahead,
  // measured the same c2 step as two -- 97.7-97.9 vs 97.3-97.6 us: the gather's tail after dense(k) comes from the
  // dense GEMMs holding the SMs' registers, not from the slot dependency)
  static constexpr int kSlots = 2;
  size_t off_tables = 0, off_flag = 0, off_x0[kSlots] = {}, off_xa = 0, off_xb = 0, off_t = 0;
  size_t off_call[kSlots] = {};  // executor per-call argument blocks (CallArgs), one per x0 slot
  std::vector<size_t> off_h;
  size_t off_idx[kSlots] = {}, off_offs[kSlots] = {}, off_dense[kSlots] = {}, off_scores[kSlots] = {};
  // runtime
  int num_sms = 148;
  bool cuda_ready = false;
  cudaEvent_t ev_embed[kSlots] = {}, ev_dense[kSlots] = {}, ev_copy[kSlots] = {};
  int64_t k = 0;
  float head_b = 0.f;  // host copy of head/b (weights are loaded synchronously)
  // tensor maps for internal A operands
  CUtensorMap tm_x0slot[kSlots], tm_xa, tm_xb, tm_t;   // A-operand / epilogue-input maps, box {64, 128}
  std::vector<CUtensorMap> tm_h;
  CUtensorMap st_xa, st_xb, st_t;                 // output (TMA store) maps, box {64, 32}
  // ensemble (config 4) buffers and maps
  struct Ens {
    // cat = [O | FFN hidden] per token: the out-projection and FFN2 become ONE GEMM with K = D + ffn
    // against [Wo | W2] (their outputs are summed anyway, A20), saving a launch and an fp32 round trip
    size_t off_S = 0, off_qkv = 0, off_cat = 0;
    std::vector<size_t> off_catW, off_catb;
    std::vector<size_t> off_qkvh, off_bqkvh;           // Wqkv / bqkv repacked head-major: head h = rows [192 h, +192)
    std::vector<CUtensorMap> Wqkvh;                    //   = [q_h | k_h | v_h] (the fused QKV + attention GEMM's B)
    CUtensorMap flat_x0[kSlots], tok_x0[kSlots], flat_xa, flat_xb, tok_xa, tok_xb, sttok_xa, sttok_xb;
    CUtensorMap st_qkv, st_hf, tm_cat;
    CUtensorMap st_S;                                  // fp32 branch sum S [B, W]: staged TMA stores (box 32 x 32)
    CUtensorMap ld_Stok;                               // the same S as tokens [B*T, D]: the FFN2 + LN input loads
    bool st_S_ok = false;
    std::vector<CUtensorMap> V, U, Wqkv, W1, Wcat;
    std::vector<CUtensorMap> V256;                     // V with 256-row boxes: t = X V^T as one-wave 128 x 256 tiles
    std::vector<CUtensorMap> W1f, W2f, Wof;            // the fused FFN's weight boxes (W1 128 rows; W2 256; Wo 128)
    CUtensorMap tok_user;
  } ens;
  // MaskNet: x0' = ReLU(W_in x0 + b_in) [B, Wp]; H = ReLU(x0' V_all^T + c_all)
  // [B, P*S*r] (every block's mask hidden comes from x0', so one GEMM covers them all);
  // block (p, q): x <- (H_pq U_pq^T + b_pq) * x, the last block of branch p writing cat[:, p*Wp ..)
  struct Mask {
    int Wp = 0, P = 0;
    size_t off_x0p = 0, off_H = 0, off_cat = 0, off_tmp[2] = {0, 0}, off_Vall = 0, off_call = 0;
    size_t off_Uall = 0, off_ball = 0;  // parallel-only (S = 1): U_p stacked [P*W', r], b_p stacked [P*W']
    CUtensorMap tm_x0p, st_x0p, st_H, tm_cat, tm_tmp[2], st_tmp[2], tmB_Vall, tmB_Uall, tm_Hall;
    std::vector<CUtensorMap> tm_Hblk, st_cat, tmB_U;
    CUtensorMap tm_cat_st;  // store map over the whole cat [B, P*W'] (grouped launch)
    int bn_proj = 0, bn_h = 0, bn_u = 0;
  } mk;
  size_t off_hpart = 0;   // split-head partial dot products [max_batch, last/256]
  int head_parts = 0;     // 0: head fused into the last MLP GEMM (last <= 256); else #256-wide parts
  std::vector<CUtensorMap> st_h;
  // CVR_GEMM_TIMELINE: per-CTA stamps of every GEMM of the last dense stage (printed at cvr_destroy)
  unsigned long long* gdbg = nullptr;
  int gdbg_n = 0;
  std::vector<int> gdbg_kid;
  // the stage being enqueued reads its batch from this per-call block (executor graphs), else nullptr
  const CallArgs* call = nullptr;
  // ---- options (cvr_set_option); every variant that measured slower in round 1 was removed
  bool pdl = true;
  int ens_u_bn = 128;       // N tile of the ensemble DCN U GEMM (option "ens_u_bn": 64 | 128)
  bool pair_ens = true;     // 2-CTA tiles for the ensemble path's GEMMs (option "pair")
  int embed_bps_pipe = 0;   // embed grid cap (CTAs/SM) in the executor; 0 = none (measured best)
  bool prefetch_b = true;
  bool f32_tma_store = true;    // option "f32_tma_store": config 4's fp32 DCN-branch output through staged TMA stores
  // option "ens_fused_attn" [1]: config 4's QKV projection + attention as one GEMM (EPI_ATTN; the qkv tensor,
  // 805 MB per layer at B = 8192, never reaches HBM).  Bit-identical to QKV GEMM + mha64; measured per layer
  // 381 us vs 257 + 247 (two epilogue groups; one group: 519 -- the attention warps' latency bounds each tile)
  bool ens_fused_attn = true;
  // option "ens_attn_tc" [1]: the fused QKV + attention GEMM with the attention itself on tcgen05 (EPI_ATTN_TC:
  // S = Q K^T and O = P V as UMMAs into the drained accumulator's TMEM columns, thread-per-row softmax from TMEM, P
  // written back to TMEM as the A operand of P V, two groups of 4 epilogue warps on alternate tiles).  Measured on
  // B200 at B = 8192: 340 us per launch vs 472 with the mma.sync core (0 = the mma.sync epilogue, EPI_ATTN); a first
  // version with P staged in shared memory and one epilogue group ran 597 us
  bool ens_attn_tc = true;
  bool ens_xv_wave = true;      // option "ens_xv_wave": config 4's t = X V^T as one wave of 128 x 256 tiles
  // option "ens_ffn_fused": config 4's FFN1 + out-projection + FFN2 + LN as one kernel (ffn_fused.cu; the hidden
  // activations never reach HBM), bit-identical to FFN1 GEMM + [O | h] GEMM with the LN epilogue
  bool ens_ffn_fused = false;
  bool zero_copy_scores = true;  // option "zero_copy_scores": cvr_score_host writes scores into pinned h_scores
  int u_bn = 192;              // option "u_bn": N tile of the low-rank U GEMM (192 when W % 192 == 0, else 64)
  int xv_bn = 0;               // option "xv_bn": N tile of t = x_l V^T (0 = by wave count, see pick_bn_xv)
  // option "epw": split epilogues 0 never, 1 always, 2 when a CTA has <= 2 tiles; default by backbone (set at create):
  // 0 for the low-rank DCN -- its MLP GEMMs then run 7-warp CTAs whose registers leave room for the next batch's
  // gather CTAs: c2's pipelined step 99.8 -> 97.6 us although the dense stage alone slows 87.0 -> 89.9 us -- and
  // 2 elsewhere (c6: 139-141 vs 142-145 us per step with 0; c4 neutral)
  int epw_mode = 2;
  bool mask_grouped = true;    // option "mask_grouped": MaskNet parallel blocks as one grouped GEMM launch
  // executor CUDA graphs: one per (stage, slot, size bucket), captured at first use and replayed for every batch
  // (the batch lives in the per-call block, so neither its pointers nor its row count are baked into the graph;
  // the bucket -- the batch size rounded up to a power of two >= 128, capped at max_batch -- only sizes the grids,
  // so a 68-item request does not launch the grids of a max_batch one)
  bool use_graphs = true;
  enum { G_EMBED = 0, G_EMBED_KEYS = 1, G_DENSE = 2, G_KINDS = 3, G_BUCKETS = 24 };
  cudaGraphExec_t gexec[G_KINDS][kSlots][G_BUCKETS] = {};
  int64_t gkernels[G_KINDS][kSlots][G_BUCKETS] = {};
  int64_t graph_captures = 0;
  void drop_graphs() {
    for (auto& kind : gexec)
      for (auto& sl : kind)
        for (auto& g : sl)
          if (g) {
            cudaGraphExecDestroy(g);
            g = nullptr;
          }
  }
  // grid size of an executor batch of `batch` rows: the next power of two >= 128, capped at max_batch
  int bucket_rows(int batch, int* idx) const {
    int b = 128, i = 0;
    while (b < batch && b < max_batch) {
      b <<= 1;
      ++i;
    }
    *idx = i;
    return b < max_batch ? b : max_batch;
  }
  std::vector<GemmPlan> plan;  // cross layers (V, U interleaved), then MLP
  // launch accounting + optional per-launch CUDA-event timing (cvr_profile_begin/end)
  int64_t launches = 0;
  // cvr_repeat_kernel: the dense stage launches only the GEMMs of role only_kid, each only_reps times
  int only_kid = -1, only_reps = 1;
  bool prof_on = false;
  size_t prof_cap = 0, prof_n = 0;
  std::vector<cudaEvent_t> prof_ev;
  std::vector<int> prof_kid;
  void pbeg(cudaStream_t s) {
    if (prof_on && prof_n < prof_cap) cudaEventRecord(prof_ev[2 * prof_n], s);
  }
  void pend(int kid, cudaStream_t s) {
    ++launches;
    if (prof_on && prof_n < prof_cap) {
      cudaEventRecord(prof_ev[2 * prof_n + 1], s);
      prof_kid[prof_n++] = kid;
    }
  }

  template <typename T = uint8_t>
  T* at(size_t off) const { return reinterpret_cast<T*>(ws + off); }
  int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    err = buf;
    return code;
  }
  int cuda_fail(cudaError_t e, const char* what) {
    return fail(CVR_E_CUDA, "%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
  }
  WSlot* slot(const std::string& n) {
    for (auto& s : wslots)
      if (s.name == n) return &s;
    return nullptr;
  }
  template <typename T = void>
  T* wptr(const std::string& n) { return reinterpret_cast<T*>(ws + slot(n)->off); }

  // ---- executor lanes (option "lanes", set before cvr_set_workspace).  With L >= 2 lanes, cvr_score /
  // cvr_score_keys / cvr_score_host deal consecutive calls round-robin over L independent pipelines of this model:
  // lane 0 is this context, lanes 1.. are full sub-contexts (their own x0 slots, intermediates, graphs, status flag
  // and weight copy) that borrow the same tables.  Every lane runs on its own pair of library streams (priorities
  // taken from the caller's streams at first use); a call's work is ordered after the caller's s_embed (inputs and
  // the scores buffer) and joined back into the caller's s_dense, so dense(k) of one lane runs beside dense(k+1) of
  // the next one: c2 86.3 vs 97.0 us per batch at L = 2 (the GEMMs of one stage leave SMs and registers idle that
  // the other stage's CTAs take); per-batch latency grows accordingly.  Everything else (cvr_embed, cvr_dense,
  // cvr_repeat_kernel, profiling) uses lane 0 on the caller's streams.
  static constexpr int kMaxLanes = 4;
  cvr_model_desc desc{};       // the creation description (arrays point into rows / mlp): sub-contexts are built from it
  int lanes = 1;
  cvr_ctx* lane_ctx[kMaxLanes] = {};  // [0] unused: lane 0 is this context
  cudaStream_t lane_se[kMaxLanes] = {}, lane_sd[kMaxLanes] = {};
  cudaEvent_t lane_in[kMaxLanes] = {}, lane_out[kMaxLanes] = {};
  int64_t lane_k = 0;
  cvr_ctx* lane(int i) { return i ? lane_ctx[i] : this; }
  const cvr_ctx* lane(int i) const { return i ? lane_ctx[i] : this; }
  size_t lane_ws_off(int i) const {  // workspace offset of lane i (each lane's share rounded to 256 B)
    size_t off = 0;
    for (int j = 0; j < i; ++j) off += j ? lane_ctx[j]->ws_need : ws_need;
    return off;
  }
};

namespace {

std::string shape_str(const std::vector<int64_t>& s) {
  std::string o = "[";
  for (size_t i = 0; i < s.size(); ++i) o += (i ? ", " : "") + std::to_string(s[i]);
  return o + "]";
}

void build_weight_slots(cvr_ctx* c) {
  auto add = [&](const std::string& n, std::vector<int64_t> sh, int dt) {
    WSlot s;
    s.name = n;
    s.shape = sh;
    s.dtype = dt;
    c->wslots.push_back(s);
  };
  const int a = c->act;
  if (c->F) {
    add("norm/mean", {c->F}, CVR_F32);
    add("norm/std", {c->F}, CVR_F32);
  }
  int prev = c->W;
  if (c->backbone == CVR_DCN_FULL) {
    for (int l = 0; l < c->n_cross; ++l) {
      add("dcn/" + std::to_string(l) + "/W", {c->W, c->W}, a);
      add("dcn/" + std::to_string(l) + "/b", {c->W}, a);
    }
  } else if (c->backbone == CVR_DCN_LOWRANK) {
    for (int l = 0; l < c->n_cross; ++l) {
      add("dcn/" + std::to_string(l) + "/V", {c->r, c->W}, a);
      add("dcn/" + std::to_string(l) + "/U", {c->W, c->r}, a);
      add("dcn/" + std::to_string(l) + "/b", {c->W}, a);
    }
  } else if (c->backbone == CVR_ENSEMBLE) {
    const int D = c->d;
    for (int l = 0; l < c->n_cross; ++l) {
      const std::string p = "ens/" + std::to_string(l) + "/";
      add(p + "dcn/V", {c->r, c->W}, a);
      add(p + "dcn/U", {c->W, c->r}, a);
      add(p + "dcn/b", {c->W}, a);
      add(p + "mha/Wqkv", {3 * D, D}, a);
      add(p + "mha/bqkv", {3 * D}, a);
      add(p + "mha/Wo", {D, D}, a);
      add(p + "mha/bo", {D}, a);
      add(p + "ffn/W1", {c->ffn, D}, a);
      add(p + "ffn/b1", {c->ffn}, a);
      add(p + "ffn/W2", {D, c->ffn}, a);
      add(p + "ffn/b2", {D}, a);
      add(p + "ln/gamma", {D}, a);
      add(p + "ln/beta", {D}, a);
    }
  }
  if (c->backbone == CVR_MASKNET) {
    const int Wp = c->mk.Wp;
    add("proj/W", {Wp, c->W}, a);
    add("proj/b", {Wp}, a);
    for (int p = 0; p < c->mk.P; ++p)
      for (int q = 0; q < c->n_cross; ++q) {
        const std::string n = "mask/" + std::to_string(p) + "/" + std::to_string(q) + "/";
        add(n + "V", {c->r, Wp}, a);
        add(n + "c", {c->r}, a);
        add(n + "U", {Wp, c->r}, a);
        add(n + "b", {Wp}, a);
      }
    prev = c->mk.P * Wp;
  }
  for (int i = 0; i < c->n_mlp; ++i) {
    add("mlp/" + std::to_string(i) + "/W", {c->mlp[i], prev}, a);
    add("mlp/" + std::to_string(i) + "/b", {c->mlp[i]}, a);
    prev = c->mlp[i];
  }
  add("head/w", {1, prev}, a);
  add("head/b", {1}, a);
}

// repacked size in the workspace
size_t packed_bytes(const cvr_ctx* c, const WSlot& s) {
  const std::string& n = s.name;
  auto ends = [&](const char* suf) { return n.size() >= strlen(suf) && n.compare(n.size() - strlen(suf), strlen(suf), suf) == 0; };
  if (c->backbone == CVR_DCN_FULL || s.shape.size() == 1 || n.rfind("norm/", 0) == 0 || n.rfind("head/", 0) == 0) {
    int64_t e = 1;
    for (auto v : s.shape) e *= v;
    if (s.shape.size() == 1 && n.rfind("dcn/", 0) == 0) e = c->x0_ld;  // padded bias
    return (size_t)e * 4;                                              // fp32 copies
  }
  if (c->backbone == CVR_ENSEMBLE) return (size_t)s.shape[0] * s.shape[1] * 2;  // W == x0_ld: no padding
  if (c->backbone == CVR_MASKNET) {  // only the projection reads x0 (padded to x0_ld)
    if (n == "proj/W") return (size_t)c->mk.Wp * c->x0_ld * 2;
    return (size_t)s.shape[0] * s.shape[1] * 2;
  }
  // bf16 GEMM operands, padded to x0_ld along W
  if (ends("/V")) return (size_t)c->r * c->x0_ld * 2;
  if (ends("/U")) return (size_t)c->x0_ld * c->r * 2;
  if (n == "mlp/0/W") return (size_t)c->mlp[0] * c->x0_ld * 2;
  return (size_t)s.shape[0] * s.shape[1] * 2;
}

int validate_desc(const cvr_model_desc* d, std::string& why) {
  char buf[256];
  auto bad = [&](const char* m) { why = m; return CVR_E_ARG; };
  if (!d) return bad("null desc");
  if (d->n_tables <= 0 || d->n_tables > 4096) return bad("n_tables out of range");
  if (!d->rows) return bad("rows is null");
  for (int t = 0; t < d->n_tables; ++t)
    if (d->rows[t] <= 0 || d->rows[t] > INT32_MAX) {
      snprintf(buf, sizeof buf, "rows[%d] out of range", t);
      why = buf;
      return CVR_E_ARG;
    }
  if (d->dim <= 0 || d->dim > 512) return bad("dim out of range");
  if (d->emb_dtype < 0 || d->emb_dtype > 2 || d->act_dtype < 0 || d->act_dtype > 1) return bad("bad dtype");
  {  // one lane group of row_bytes / 16 lanes per bag: 2, 4, 8, 16 or 32 lanes (a power of two, embed.cu)
    const int lanes = d->dim * (int)elt_size(d->emb_dtype) / 16;
    if ((d->dim * (int)elt_size(d->emb_dtype)) % 16 != 0 || lanes < 2 || lanes > 32 || (lanes & (lanes - 1)))
      return bad("dim * sizeof(row element) must be 32, 64, 128, 256 or 512 bytes");
  }
  if (d->n_dense < 0 || d->n_cross < 0 || d->n_cross > kMaxLayers || d->n_mlp < 1 || d->n_mlp > kMaxLayers)
    return bad("layer counts out of range");
  if (!d->mlp_dims) return bad("mlp_dims is null");
  for (int i = 0; i < d->n_mlp; ++i)
    if (d->mlp_dims[i] <= 0) return bad("mlp_dims must be positive");
  if (d->max_batch <= 0 || d->max_nnz < 0) return bad("max_batch / max_nnz out of range");
  if (d->world_size < 1 || d->rank < 0 || d->rank >= d->world_size) return bad("bad world_size / rank");
  if (d->backbone == CVR_DCN_FULL) {
    if (d->act_dtype != CVR_F32) return bad("DCN_FULL runs the fp32 path: act_dtype must be CVR_F32");
  } else if (d->backbone == CVR_DCN_LOWRANK) {
    if (d->act_dtype != CVR_BF16) return bad("DCN_LOWRANK runs the bf16 tensor-core path: act_dtype must be CVR_BF16");
    if (d->cross_rank <= 0 || d->cross_rank % 64) return bad("cross_rank must be a positive multiple of 64");
    for (int i = 0; i < d->n_mlp; ++i)
      if (d->mlp_dims[i] % 64) return bad("mlp_dims must be multiples of 64 on the bf16 path");
    const int last = d->mlp_dims[d->n_mlp - 1];
    if (!(last == 64 || last == 128 || last == 256 || last % 256 == 0))
      return bad("last MLP width must be 64, 128, 256 (fused head) or a multiple of 256 (split head)");
  } else if (d->backbone == CVR_ENSEMBLE) {
    if (d->act_dtype != CVR_BF16) return bad("ENSEMBLE runs the bf16 tensor-core path: act_dtype must be CVR_BF16");
    if (d->n_heads != 4 || d->dim != 256)
      return bad("ensemble layer: 4 heads x 64 over tokens of dim 256 (BASELINE.json configs[3], A20)");
    if (d->n_tables != 64)  // the attention kernels hold one example's 64 tokens per 64-row block (S = 64)
      return bad("ensemble layer: the attention runs over exactly 64 tokens (n_tables = 64, BASELINE.json configs[3])");
    if (d->n_dense != 0) return bad("ensemble: the tokens are the pooled tables, no dense features (A20)");
    if (d->cross_rank <= 0 || d->cross_rank % 128) return bad("ensemble cross_rank must be a multiple of 128");
    if (d->ffn_dim <= 0 || d->ffn_dim % 128) return bad("ffn_dim must be a multiple of 128");
    for (int i = 0; i + 1 < d->n_mlp; ++i)
      if (d->mlp_dims[i] % 128) return bad("hidden MLP widths must be multiples of 128 on the ensemble path");
    const int last = d->mlp_dims[d->n_mlp - 1];
    if (!(last == 64 || last == 128 || last == 256 || last % 256 == 0)) return bad("last MLP width: 64/128/256 or k*256");
  } else if (d->backbone == CVR_MASKNET) {
    if (d->act_dtype != CVR_BF16) return bad("MASKNET runs the bf16 tensor-core path: act_dtype must be CVR_BF16");
    if (d->cross_width <= 0 || d->cross_width % 128) return bad("MASKNET cross_width must be a positive multiple of 128");
    if (d->cross_rank <= 0 || d->cross_rank % 64) return bad("MASKNET cross_rank (mask hidden width) must be a multiple of 64");
    if (d->n_parallel < 1 || d->n_parallel > 8 || d->n_cross < 1) return bad("MASKNET needs n_parallel in [1, 8], n_cross >= 1");
    for (int i = 0; i < d->n_mlp; ++i)
      if (d->mlp_dims[i] % 64) return bad("mlp_dims must be multiples of 64 on the bf16 path");
    const int last = d->mlp_dims[d->n_mlp - 1];
    if (!(last == 64 || last == 128 || last == 256 || last % 256 == 0))
      return bad("last MLP width must be 64, 128, 256 (fused head) or a multiple of 256 (split head)");
  } else {
    return CVR_E_UNSUPPORTED;
  }
  return CVR_OK;
}

size_t carve(size_t& cur, size_t bytes) {
  const size_t o = (cur + 255) & ~size_t(255);
  cur = o + bytes;
  return o;
}

// N-tile width: wide tiles halve the bytes ingested per FLOP (measured: 4096x1024x1728 13.5 us at BN=256
// vs 16.2 at 128), as long as enough tiles remain to cover the SMs.
int pick_bn(int N, int64_t M = 0) {
  const int64_t mt = (M + 127) / 128;
  if (N % 256 == 0 && N > 256 && mt * (N / 256) >= 100) return 256;
  if (N > 256 && N % 128 == 0) return 128;
  return 64;
}

// N tile of t = x_l V^T (N = r, small): pick the tile minimising waves x k-block cost.  Measured per 128 x BN x 64
// k-block on B200 (per-SM ingest / small-N MMA bound): ~211 ns at BN = 64, ~280 ns at 256 -- 64-wide tiles
// win while they fit one wave (c2: 128 tiles), full-width tiles once the row blocks alone fill the SMs.
int pick_bn_xv(int N, int64_t M, int num_sms) {
  const int64_t mt = (M + 127) / 128;
  double best = 1e30;
  int bn = 64;
  const int cand[3] = {64, 128, 256};
  const double cost[3] = {211, 240, 280};
  for (int i = 0; i < 3; ++i) {
    if (N % cand[i]) continue;
    const int64_t tiles = mt * (N / cand[i]);
    const double t = (double)((tiles + num_sms - 1) / num_sms) * cost[i];
    if (t < best - 1e-9) {
      best = t;
      bn = cand[i];
    }
  }
  return bn;
}

}  // namespace

extern "C" {

const char* cvr_version(void) { return "cvr 0.1 (sm_100a)"; }

const char* cvr_status_string(int s) {
  switch (s) {
    case CVR_OK: return "CVR_OK";
    case CVR_E_ARG: return "CVR_E_ARG";
    case CVR_E_SHAPE: return "CVR_E_SHAPE";
    case CVR_E_DTYPE: return "CVR_E_DTYPE";
    case CVR_E_STATE: return "CVR_E_STATE";
    case CVR_E_INDEX: return "CVR_E_INDEX";
    case CVR_E_NOMEM: return "CVR_E_NOMEM";
    case CVR_E_CUDA: return "CVR_E_CUDA";
    case CVR_E_NCCL: return "CVR_E_NCCL";
    case CVR_E_OVERLOAD: return "CVR_E_OVERLOAD";
    case CVR_E_UNSUPPORTED: return "CVR_E_UNSUPPORTED";
  }
  return "CVR_E_?";
}

int cvr_create(const cvr_model_desc* desc, cvr_ctx** out) {
  if (!out) return CVR_E_ARG;
  *out = nullptr;
  std::string why;
  int st = validate_desc(desc, why);
  cvr_ctx* c = new cvr_ctx();
  if (st != CVR_OK) {
    c->err = why.empty() ? "unsupported model description" : why;
    *out = c;  // returned so the caller can read cvr_last_error, then must destroy it
    return st;
  }
  c->desc = *desc;
  c->T = desc->n_tables;
  c->rows.assign(desc->rows, desc->rows + c->T);
  c->d = desc->dim;
  c->emb_dtype = desc->emb_dtype;
  c->F = desc->n_dense;
  c->act = desc->act_dtype;
  c->backbone = desc->backbone;
  c->n_cross = desc->n_cross;
  c->r = desc->cross_rank;
  c->n_mlp = desc->n_mlp;
  c->mlp.assign(desc->mlp_dims, desc->mlp_dims + c->n_mlp);
  c->desc.rows = c->rows.data();
  c->desc.mlp_dims = c->mlp.data();
  c->n_heads = desc->n_heads;
  c->ffn = desc->ffn_dim;
  c->max_batch = desc->max_batch;
  c->max_nnz = desc->max_nnz;
  c->world = desc->world_size;
  c->rank = desc->rank;
  c->W = c->T * c->d + c->F;
  if (c->backbone == CVR_MASKNET) {
    c->mk.Wp = desc->cross_width;
    c->mk.P = desc->n_parallel;
  }
  c->epw_mode = c->backbone == CVR_DCN_LOWRANK ? 0 : 2;
  c->x0_ld = c->act == CVR_F32 ? round_up(c->W, 4) : round_up(c->W, 64);
  for (int t = 0; t < c->T; ++t)
    if (t % c->world == c->rank) c->local_tables.push_back(t);
  c->T_pad = (c->T + c->world - 1) / c->world;
  c->htables.resize(c->local_tables.size());
  c->tvocab.assign(c->T, 0);
  c->tmean.assign(c->T, 0);
  build_weight_slots(c);

  // ---- workspace layout
  size_t cur = 0;
  for (auto& s : c->wslots) {
    s.bytes = packed_bytes(c, s);
    s.off = carve(cur, s.bytes);
  }
  const size_t ae = elt_size(c->act);
  const int64_t B = c->max_batch;
  c->off_tables = carve(cur, sizeof(TableDesc) * std::max<size_t>(1, c->local_tables.size()));
  c->off_flag = carve(cur, 256);
  for (int i = 0; i < cvr_ctx::kSlots; ++i) c->off_call[i] = carve(cur, sizeof(CallArgs));
  if (c->world > 1) c->off_peers = carve(cur, (size_t)4 * c->world * sizeof(void*));
  for (int i = 0; i < cvr_ctx::kSlots; ++i) c->off_x0[i] = carve(cur, (size_t)B * c->x0_ld * ae);
  if (c->backbone == CVR_DCN_LOWRANK) {
    c->off_xa = carve(cur, (size_t)B * c->x0_ld * 2);
    c->off_xb = carve(cur, (size_t)B * c->x0_ld * 2);
    c->off_t = carve(cur, (size_t)B * c->r * 2);
    for (int i = 0; i + 1 < c->n_mlp; ++i) c->off_h.push_back(carve(cur, (size_t)B * c->mlp[i] * 2));
  } else if (c->backbone == CVR_ENSEMBLE) {
    const int64_t BT = B * c->T;  // tokens
    c->off_xa = carve(cur, (size_t)B * c->x0_ld * 2);
    c->off_xb = carve(cur, (size_t)B * c->x0_ld * 2);
    c->off_t = carve(cur, (size_t)B * c->r * 2);
    c->ens.off_S = carve(cur, (size_t)B * c->x0_ld * 4);
    c->ens.off_qkv = carve(cur, (size_t)BT * 3 * c->d * 2);
    c->ens.off_cat = carve(cur, (size_t)BT * (c->d + c->ffn) * 2);
    for (int l = 0; l < c->n_cross; ++l) {
      c->ens.off_catW.push_back(carve(cur, (size_t)c->d * (c->d + c->ffn) * 2));
      c->ens.off_catb.push_back(carve(cur, (size_t)c->d * 4));
      c->ens.off_qkvh.push_back(carve(cur, (size_t)3 * c->d * c->d * 2));
      c->ens.off_bqkvh.push_back(carve(cur, (size_t)3 * c->d * 4));
    }
    for (int i = 0; i + 1 < c->n_mlp; ++i) c->off_h.push_back(carve(cur, (size_t)B * c->mlp[i] * 2));
  } else if (c->backbone == CVR_MASKNET) {
    auto& K = c->mk;
    const int nb = K.P * c->n_cross;
    K.off_x0p = carve(cur, (size_t)B * K.Wp * 2);
    K.off_H = carve(cur, (size_t)B * nb * c->r * 2);
    K.off_cat = carve(cur, (size_t)B * K.P * K.Wp * 2);
    if (c->n_cross > 1)
      for (int i = 0; i < 2; ++i) K.off_tmp[i] = carve(cur, (size_t)B * K.Wp * 2);
    K.off_Vall = carve(cur, (size_t)nb * c->r * K.Wp * 2);
    K.off_call = carve(cur, (size_t)nb * c->r * 4);
    if (c->n_cross == 1) {
      K.off_Uall = carve(cur, (size_t)K.P * K.Wp * c->r * 2);
      K.off_ball = carve(cur, (size_t)K.P * K.Wp * 4);
    }
    for (int i = 0; i + 1 < c->n_mlp; ++i) c->off_h.push_back(carve(cur, (size_t)B * c->mlp[i] * 2));
  }
  if (c->backbone != CVR_DCN_FULL) {
    const int last = c->mlp[c->n_mlp - 1];
    c->head_parts = (last == 64 || last == 128 || last == 256) ? 0 : last / 256;
    if (c->head_parts) c->off_hpart = carve(cur, (size_t)B * c->head_parts * 4);
  }
  const int64_t Bin = c->world > 1 ? B * c->world : B;  // sharded: indices cover the global batch
  const int T_l = (int)c->local_tables.size();
  for (int i = 0; i < cvr_ctx::kSlots; ++i) {
    c->off_idx[i] = carve(cur, (size_t)std::max<int64_t>(c->max_nnz, 1) * 4);
    c->off_offs[i] = carve(cur, (size_t)(T_l * Bin + 1) * 4);
    c->off_dense[i] = carve(cur, (size_t)B * std::max(c->F, 1) * 4);
    c->off_scores[i] = carve(cur, (size_t)B * 4);
  }
  c->ws_need = (cur + 255) & ~size_t(255);
  *out = c;
  return CVR_OK;
}

int cvr_destroy(cvr_ctx* c) {
  if (!c) return CVR_E_ARG;
  if (c->lanes > 1) cudaDeviceSynchronize();  // the lanes' streams may still run work of this context
  for (int i = 1; i < cvr_ctx::kMaxLanes; ++i)
    if (c->lane_ctx[i]) cvr_destroy(c->lane_ctx[i]);
  for (int i = 0; i < cvr_ctx::kMaxLanes; ++i) {
    if (c->lane_se[i]) cudaStreamDestroy(c->lane_se[i]);
    if (c->lane_sd[i]) cudaStreamDestroy(c->lane_sd[i]);
    if (c->lane_in[i]) cudaEventDestroy(c->lane_in[i]);
    if (c->lane_out[i]) cudaEventDestroy(c->lane_out[i]);
  }
  if (c->gdbg) {  // debug: GEMM timeline of the last dense stage (us from the first GEMM's first CTA entry)
    std::vector<unsigned long long> h((size_t)32 * 160 * 8);
    cudaDeviceSynchronize();
    cudaMemcpy(h.data(), c->gdbg, h.size() * 8, cudaMemcpyDeviceToHost);
    const int n = std::min<int>((int)c->gdbg_kid.size(), 32);
    unsigned long long t0 = ~0ull;
    for (int b = 0; b < 160; ++b)
      if (h[(size_t)b * 8]) t0 = std::min(t0, h[(size_t)b * 8]);
    const char* nm[8] = {"entry", "deps", "1st-stage", "last-mma", "1st-acc", "epi-done", "exit", ""};
    for (int g = 0; g < n; ++g) {
      fprintf(stderr, "gemm %2d %-16s", g, kKernelNames[c->gdbg_kid[g]]);
      for (int i = 0; i < 7; ++i) {
        double mn = 1e30, mx = 0;
        for (int b = 0; b < 160; ++b) {
          const unsigned long long v = h[((size_t)g * 160 + b) * 8 + i];
          if (!v) continue;
          mn = std::min(mn, (double)(v - t0) / 1e3);
          mx = std::max(mx, (double)(v - t0) / 1e3);
        }
        fprintf(stderr, " %s %.2f-%.2f", nm[i], mn, mx);
      }
      fprintf(stderr, "\n");
    }
    cudaFree(c->gdbg);
  }
  for (auto ev : c->prof_ev) cudaEventDestroy(ev);
  c->drop_graphs();
  if (c->nccl_comm && g_nccl.dl) g_nccl.commDestroy(c->nccl_comm);
  for (int i = 0; i < cvr_ctx::kSlots; ++i) {
    if (c->ev_embed[i]) cudaEventDestroy(c->ev_embed[i]);
    if (c->ev_dense[i]) cudaEventDestroy(c->ev_dense[i]);
    if (c->ev_copy[i]) cudaEventDestroy(c->ev_copy[i]);
  }
  delete c;
  return CVR_OK;
}

const char* cvr_last_error(const cvr_ctx* c) { return c ? c->err.c_str() : "null ctx"; }

int cvr_workspace_bytes(const cvr_ctx* c, size_t* bytes) {
  if (!c || !bytes) return CVR_E_ARG;
  *bytes = c->lane_ws_off(c->lanes);  // every lane's share (ws_need alone at one lane)
  return CVR_OK;
}

int cvr_x0_layout(const cvr_ctx* c, int* ld, int* dt) {
  if (!c || !ld || !dt) return CVR_E_ARG;
  *ld = (int)c->x0_ld;
  *dt = c->act;
  return CVR_OK;
}

// a new lane starts with its parent's options (options set later are forwarded by cvr_set_option)
static void copy_options(cvr_ctx* t, const cvr_ctx* c) {
  t->pdl = c->pdl;
  t->ens_u_bn = c->ens_u_bn;
  t->pair_ens = c->pair_ens;
  t->embed_bps_pipe = c->embed_bps_pipe;
  t->prefetch_b = c->prefetch_b;
  t->f32_tma_store = c->f32_tma_store;
  t->ens_fused_attn = c->ens_fused_attn;
  t->ens_attn_tc = c->ens_attn_tc;
  t->ens_xv_wave = c->ens_xv_wave;
  t->ens_ffn_fused = c->ens_ffn_fused;
  t->zero_copy_scores = c->zero_copy_scores;
  t->u_bn = c->u_bn;
  t->xv_bn = c->xv_bn;
  t->epw_mode = c->epw_mode;
  t->mask_grouped = c->mask_grouped;
  t->use_graphs = c->use_graphs;
  t->tvocab = c->tvocab;
  t->tmean = c->tmean;
  t->any_mean = c->any_mean;
}

// apply the same call to every sub-context lane (1..lanes-1) first; lc_ names the lane inside `call_expr`
#define CVR_FORWARD_LANES(c, call_expr)                                                 \
  for (int li_ = 1; li_ < (c)->lanes; ++li_) {                                         \
    cvr_ctx* lc_ = (c)->lane_ctx[li_];                                                 \
    const int st_ = (call_expr);                                                       \
    if (st_ != CVR_OK) return (c)->fail(st_, "lane %d: %s", li_, lc_->err.c_str());   \
  }

static int set_workspace_one(cvr_ctx* c, void* d_ws, size_t bytes);

int cvr_set_workspace(cvr_ctx* c, void* d_ws, size_t bytes) {
  if (!c || !d_ws) return CVR_E_ARG;
  if (reinterpret_cast<uintptr_t>(d_ws) & 255) return c->fail(CVR_E_ARG, "workspace must be 256-byte aligned");
  const size_t need = c->lane_ws_off(c->lanes);
  if (bytes < need) return c->fail(CVR_E_NOMEM, "workspace %zu bytes < required %zu", bytes, need);
  for (int i = c->lanes - 1; i >= 0; --i) {  // lane 0 (this context) last: its state is what callers inspect
    cvr_ctx* t = c->lane(i);
    const int st = set_workspace_one(t, reinterpret_cast<uint8_t*>(d_ws) + c->lane_ws_off(i), t->ws_need);
    if (st != CVR_OK) return i ? c->fail(st, "lane %d: %s", i, t->err.c_str()) : st;
  }
  return CVR_OK;
}

static int set_workspace_one(cvr_ctx* c, void* d_ws, size_t bytes) {
  if (bytes < c->ws_need) return c->fail(CVR_E_NOMEM, "workspace %zu bytes < required %zu", bytes, c->ws_need);
  c->ws = reinterpret_cast<uint8_t*>(d_ws);
  c->ws_bytes = bytes;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, dev);
  for (int i = 0; i < cvr_ctx::kSlots && e == cudaSuccess; ++i) {
    if (!c->ev_embed[i]) e = cudaEventCreateWithFlags(&c->ev_embed[i], cudaEventDisableTiming);
    if (e == cudaSuccess && !c->ev_dense[i]) e = cudaEventCreateWithFlags(&c->ev_dense[i], cudaEventDisableTiming);
    if (e == cudaSuccess && !c->ev_copy[i]) e = cudaEventCreateWithFlags(&c->ev_copy[i], cudaEventDisableTiming);
  }
  if (e == cudaSuccess) e = cudaMemset(c->ws + c->off_flag, 0, 256);
  // zero the activation slots once so padding columns / tail rows are defined
  if (e == cudaSuccess) e = cudaMemset(c->ws + c->off_x0[0], 0, c->ws_need - c->off_x0[0]);
  if (e != cudaSuccess) return c->cuda_fail(e, "cvr_set_workspace");
  if (getenv("CVR_GEMM_TIMELINE") && !c->gdbg) {
    cudaMalloc(&c->gdbg, (size_t)32 * 160 * 8 * 8);
    cudaMemset(c->gdbg, 0, (size_t)32 * 160 * 8 * 8);
  }
  c->cuda_ready = true;
  c->k = 0;
  c->drop_graphs();
  c->weights_loaded = false;
  for (auto& s : c->wslots) s.loaded = false;
  if (c->backbone == CVR_DCN_LOWRANK) {
    const char* er = nullptr;
    const int64_t B = c->max_batch;
    bool ok = true;
    for (int i = 0; i < cvr_ctx::kSlots; ++i) {
      ok &= encode_tmap_bf16(&c->tm_x0slot[i], c->ws + c->off_x0[i], B, c->x0_ld, c->x0_ld, 128, &er) == 0;
    }
    ok &= encode_tmap_bf16(&c->tm_xa, c->ws + c->off_xa, B, c->x0_ld, c->x0_ld, 128, &er) == 0;
    ok &= encode_tmap_bf16(&c->tm_xb, c->ws + c->off_xb, B, c->x0_ld, c->x0_ld, 128, &er) == 0;
    ok &= encode_tmap_bf16(&c->tm_t, c->ws + c->off_t, B, c->r, c->r, 128, &er) == 0;
    ok &= encode_tmap_bf16(&c->st_xa, c->ws + c->off_xa, B, c->x0_ld, c->x0_ld, 32, &er) == 0;
    ok &= encode_tmap_bf16(&c->st_xb, c->ws + c->off_xb, B, c->x0_ld, c->x0_ld, 32, &er) == 0;
    ok &= encode_tmap_bf16(&c->st_t, c->ws + c->off_t, B, c->r, c->r, 32, &er) == 0;
    c->tm_h.resize(c->off_h.size());
    c->st_h.resize(c->off_h.size());
    for (size_t i = 0; i < c->off_h.size(); ++i) {
      ok &= encode_tmap_bf16(&c->tm_h[i], c->ws + c->off_h[i], B, c->mlp[i], c->mlp[i], 128, &er) == 0;
      ok &= encode_tmap_bf16(&c->st_h[i], c->ws + c->off_h[i], B, c->mlp[i], c->mlp[i], 32, &er) == 0;
    }
    if (!ok) return c->fail(CVR_E_CUDA, "tensor map encode: %s", er ? er : "?");
  }
  if (c->backbone == CVR_MASKNET) {
    const char* er = nullptr;
    const int64_t B = c->max_batch;
    auto& K = c->mk;
    const int nb = K.P * c->n_cross, HW = nb * c->r, CW = K.P * K.Wp;
    bool ok = true;
    for (int i = 0; i < cvr_ctx::kSlots; ++i) {
      ok &= encode_tmap_bf16(&c->tm_x0slot[i], c->ws + c->off_x0[i], B, c->x0_ld, c->x0_ld, 128, &er) == 0;
    }
    ok &= encode_tmap_bf16(&K.tm_x0p, c->ws + K.off_x0p, B, K.Wp, K.Wp, 128, &er) == 0;
    ok &= encode_tmap_bf16(&K.st_x0p, c->ws + K.off_x0p, B, K.Wp, K.Wp, 32, &er) == 0;
    ok &= encode_tmap_bf16(&K.st_H, c->ws + K.off_H, B, HW, HW, 32, &er) == 0;
    K.tm_Hblk.assign(nb, CUtensorMap{});
    for (int j = 0; j < nb; ++j)  // the r columns of block j inside H (row stride P*S*r)
      ok &= encode_tmap_bf16(&K.tm_Hblk[j], c->ws + K.off_H + (size_t)j * c->r * 2, B, c->r, HW, 128, &er) == 0;
    ok &= encode_tmap_bf16(&K.tm_cat, c->ws + K.off_cat, B, CW, CW, 128, &er) == 0;
    ok &= encode_tmap_bf16(&K.tm_cat_st, c->ws + K.off_cat, B, CW, CW, 32, &er) == 0;
    K.st_cat.assign(K.P, CUtensorMap{});
    for (int p = 0; p < K.P; ++p)
      ok &= encode_tmap_bf16(&K.st_cat[p], c->ws + K.off_cat + (size_t)p * K.Wp * 2, B, K.Wp, CW, 32, &er) == 0;
    if (c->n_cross > 1)
      for (int i = 0; i < 2; ++i) {
        ok &= encode_tmap_bf16(&K.tm_tmp[i], c->ws + K.off_tmp[i], B, K.Wp, K.Wp, 128, &er) == 0;
        ok &= encode_tmap_bf16(&K.st_tmp[i], c->ws + K.off_tmp[i], B, K.Wp, K.Wp, 32, &er) == 0;
      }
    c->tm_h.resize(c->off_h.size());
    c->st_h.resize(c->off_h.size());
    for (size_t i = 0; i < c->off_h.size(); ++i) {
      ok &= encode_tmap_bf16(&c->tm_h[i], c->ws + c->off_h[i], B, c->mlp[i], c->mlp[i], 128, &er) == 0;
      ok &= encode_tmap_bf16(&c->st_h[i], c->ws + c->off_h[i], B, c->mlp[i], c->mlp[i], 32, &er) == 0;
    }
    if (!ok) return c->fail(CVR_E_CUDA, "tensor map encode: %s", er ? er : "?");
  }
  if (c->backbone == CVR_ENSEMBLE) {
    const char* er = nullptr;
    const int64_t B = c->max_batch, BT = B * c->T, D = c->d, W = c->x0_ld;
    auto& E = c->ens;
    bool ok = true;
    for (int i = 0; i < cvr_ctx::kSlots; ++i) {
      ok &= encode_tmap_bf16(&E.flat_x0[i], c->ws + c->off_x0[i], B, W, W, 128, &er) == 0;
      ok &= encode_tmap_bf16(&E.tok_x0[i], c->ws + c->off_x0[i], BT, D, D, 128, &er) == 0;
    }
    ok &= encode_tmap_bf16(&E.flat_xa, c->ws + c->off_xa, B, W, W, 128, &er) == 0;
    ok &= encode_tmap_bf16(&E.flat_xb, c->ws + c->off_xb, B, W, W, 128, &er) == 0;
    ok &= encode_tmap_bf16(&E.tok_xa, c->ws + c->off_xa, BT, D, D, 128, &er) == 0;
    ok &= encode_tmap_bf16(&E.tok_xb, c->ws + c->off_xb, BT, D, D, 128, &er) == 0;
    ok &= encode_tmap_bf16(&E.sttok_xa, c->ws + c->off_xa, BT, D, D, 32, &er) == 0;
    ok &= encode_tmap_bf16(&E.sttok_xb, c->ws + c->off_xb, BT, D, D, 32, &er) == 0;
    ok &= encode_tmap_bf16(&c->tm_t, c->ws + c->off_t, B, c->r, c->r, 128, &er) == 0;
    ok &= encode_tmap_bf16(&c->st_t, c->ws + c->off_t, B, c->r, c->r, 32, &er) == 0;
    ok &= encode_tmap_bf16(&E.st_qkv, c->ws + E.off_qkv, BT, 3 * D, 3 * D, 32, &er) == 0;
    E.st_S_ok = encode_tmap_f32_store(&E.st_S, c->ws + E.off_S, B, W, W, &er) == 0 &&
                encode_tmap_f32_store(&E.ld_Stok, c->ws + E.off_S, BT, D, D, &er) == 0;
    ok &= E.st_S_ok;
    const int64_t CW = D + c->ffn;
    ok &= encode_tmap_bf16(&E.st_hf, c->ws + E.off_cat + D * 2, BT, c->ffn, CW, 32, &er) == 0;
    ok &= encode_tmap_bf16(&E.tm_cat, c->ws + E.off_cat, BT, CW, CW, 128, &er) == 0;
    c->tm_h.resize(c->off_h.size());
    c->st_h.resize(c->off_h.size());
    for (size_t i = 0; i < c->off_h.size(); ++i) {
      ok &= encode_tmap_bf16(&c->tm_h[i], c->ws + c->off_h[i], B, c->mlp[i], c->mlp[i], 128, &er) == 0;
      ok &= encode_tmap_bf16(&c->st_h[i], c->ws + c->off_h[i], B, c->mlp[i], c->mlp[i], 32, &er) == 0;
    }
    if (!ok) return c->fail(CVR_E_CUDA, "tensor map encode: %s", er ? er : "?");
  }
  return CVR_OK;
}

int cvr_load_tables(cvr_ctx* c, int n, const int* ids, const void* const* d_rows, const int64_t* strides) {
  if (!c || !ids || !d_rows || !strides) return CVR_E_ARG;
  CVR_FORWARD_LANES(c, cvr_load_tables(lc_, n, ids, d_rows, strides));
  if (!c->cuda_ready) return c->fail(CVR_E_STATE, "cvr_load_tables before cvr_set_workspace");
  if (n != (int)c->local_tables.size())
    return c->fail(CVR_E_SHAPE, "expected %zu tables for rank %d, got %d", c->local_tables.size(), c->rank, n);
  const int64_t row_bytes = (int64_t)c->d * elt_size(c->emb_dtype);
  for (int i = 0; i < n; ++i) {
    if (ids[i] != c->local_tables[i])
      return c->fail(CVR_E_SHAPE, "table slot %d: expected table id %d, got %d", i, c->local_tables[i], ids[i]);
    if (!d_rows[i]) return c->fail(CVR_E_ARG, "table %d: null pointer", ids[i]);
    if ((reinterpret_cast<uintptr_t>(d_rows[i]) & 15) || (strides[i] & 15) || strides[i] < row_bytes)
      return c->fail(CVR_E_ARG, "table %d: base and row stride must be 16-byte aligned, stride >= %lld", ids[i],
                     (long long)row_bytes);
    const int64_t v = c->tvocab[ids[i]];
    c->htables[i] = TableDesc{reinterpret_cast<const uint8_t*>(d_rows[i]), strides[i], c->rows[ids[i]], v,
                              v > 0 ? ~0ull / (uint64_t)v : 0ull, c->tmean[ids[i]]};
  }
  cudaError_t e = cudaMemcpy(c->ws + c->off_tables, c->htables.data(), sizeof(TableDesc) * n, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return c->cuda_fail(e, "cvr_load_tables");
  c->tables_loaded = true;
  return CVR_OK;
}

namespace {

int encode_plan(cvr_ctx* c) {
  c->plan.clear();
  const char* er = nullptr;
  auto addp = [&](const std::string& wn, int N, int K, int BN, Epi epi) -> bool {
    GemmPlan g;
    g.N = N;
    g.K = K;
    g.BN = BN;
    g.epi = epi;
    if (encode_tmap_bf16(&g.tmB, c->wptr(wn), N, K, K, BN, &er) != 0) return false;
    c->plan.push_back(g);
    return true;
  };
  bool ok = true;
  for (int l = 0; l < c->n_cross; ++l) {
    const int bn_v = c->xv_bn ? c->xv_bn : pick_bn_xv(c->r, c->max_batch, c->num_sms > 0 ? c->num_sms : 148);
    ok &= addp("dcn/" + std::to_string(l) + "/V", c->r, (int)c->x0_ld, bn_v, EPI_STORE);
    // U GEMM: 192-wide tiles (EIN-ring epilogue) when W allows -- 1/3 of the t re-reads of 64-wide tiles
    // (measured 4096x1728x256: 7.4 us at BN = 192 vs 10.3 at 64)
    const bool u192 = c->u_bn == 192 && c->x0_ld % 192 == 0;
    ok &= addp("dcn/" + std::to_string(l) + "/U", (int)c->x0_ld, c->r, u192 ? 192 : pick_bn((int)c->x0_ld), EPI_CROSS);
  }
  int K = (int)c->x0_ld;
  for (int i = 0; i < c->n_mlp; ++i) {
    const bool last = i + 1 == c->n_mlp;
    const int bn = last ? (c->head_parts ? 256 : c->mlp[i]) : pick_bn(c->mlp[i], c->max_batch);
    const Epi ep = last ? (c->head_parts ? EPI_HEAD_PARTIAL : EPI_HEAD) : EPI_BIAS_RELU;
    ok &= addp("mlp/" + std::to_string(i) + "/W", c->mlp[i], K, bn, ep);
    K = c->mlp[i];
  }
  if (!ok) return c->fail(CVR_E_CUDA, "tensor map encode: %s", er ? er : "?");
  return CVR_OK;
}

int encode_plan_ensemble(cvr_ctx* c) {
  const char* er = nullptr;
  auto& E = c->ens;
  const int D = c->d, W = (int)c->x0_ld, r = c->r, F = c->ffn;
  E.V.assign(c->n_cross, {});
  E.U.assign(c->n_cross, {});
  E.Wqkv.assign(c->n_cross, {});
  E.Wqkvh.assign(c->n_cross, {});
  E.V256.assign(c->n_cross, {});
  E.W1.assign(c->n_cross, {});
  E.Wcat.assign(c->n_cross, {});
  E.W1f.assign(c->n_cross, {});
  E.W2f.assign(c->n_cross, {});
  E.Wof.assign(c->n_cross, {});
  bool ok = true;
  for (int l = 0; l < c->n_cross; ++l) {
    const std::string p = "ens/" + std::to_string(l) + "/";
    const int dv = c->pair_ens ? 2 : 1;  // B boxes hold BN/2 rows per CTA of a pair
    ok &= encode_tmap_bf16(&E.V[l], c->wptr(p + "dcn/V"), r, W, W, 128 / dv, &er) == 0;
    if (r % 256 == 0) ok &= encode_tmap_bf16(&E.V256[l], c->wptr(p + "dcn/V"), r, W, W, 256, &er) == 0;
    ok &= encode_tmap_bf16(&E.U[l], c->wptr(p + "dcn/U"), W, r, r, c->ens_u_bn / dv, &er) == 0;
    ok &= encode_tmap_bf16(&E.Wqkv[l], c->wptr(p + "mha/Wqkv"), 3 * D, D, D, 256 / dv, &er) == 0;
    ok &= encode_tmap_bf16(&E.W1[l], c->wptr(p + "ffn/W1"), F, D, D, 256 / dv, &er) == 0;
    // [Wo | W2] and bo + b2, assembled in the workspace from the loaded copies
    cudaError_t e1 = cudaMemcpy2D(c->ws + E.off_catW[l], (size_t)(D + F) * 2, c->wptr(p + "mha/Wo"), (size_t)D * 2,
                                  (size_t)D * 2, D, cudaMemcpyDeviceToDevice);
    cudaError_t e2 = cudaMemcpy2D(c->ws + E.off_catW[l] + (size_t)D * 2, (size_t)(D + F) * 2, c->wptr(p + "ffn/W2"),
                                  (size_t)F * 2, (size_t)F * 2, D, cudaMemcpyDeviceToDevice);
    std::vector<float> bo(D), b2(D);
    cudaError_t e3 = cudaMemcpy(bo.data(), c->wptr(p + "mha/bo"), D * 4, cudaMemcpyDeviceToHost);
    cudaError_t e4 = cudaMemcpy(b2.data(), c->wptr(p + "ffn/b2"), D * 4, cudaMemcpyDeviceToHost);
    for (int i = 0; i < D; ++i) bo[i] += b2[i];
    cudaError_t e5 = cudaMemcpy(c->ws + E.off_catb[l], bo.data(), D * 4, cudaMemcpyHostToDevice);
    if (e1 || e2 || e3 || e4 || e5) return c->fail(CVR_E_CUDA, "assembling [Wo | W2]");
    ok &= encode_tmap_bf16(&E.Wcat[l], c->ws + E.off_catW[l], D, D + F, D + F, 256 / dv, &er) == 0;
    ok &= encode_tmap_bf16(&E.W1f[l], c->wptr(p + "ffn/W1"), F, D, D, 128, &er) == 0;
    ok &= encode_tmap_bf16(&E.W2f[l], c->ws + E.off_catW[l], D, D + F, D + F, 256, &er) == 0;
    ok &= encode_tmap_bf16(&E.Wof[l], c->ws + E.off_catW[l], D, D + F, D + F, 128, &er) == 0;
    // head-major [q_h | k_h | v_h] copies of Wqkv / bqkv for the fused QKV + attention GEMM (EPI_ATTN)
    if (D == 64 * c->n_heads) {
      std::vector<float> bq(3 * D), bh(3 * D);
      cudaError_t e6 = cudaMemcpy(bq.data(), c->wptr(p + "mha/bqkv"), 3 * D * 4, cudaMemcpyDeviceToHost);
      for (int h = 0; h < c->n_heads && e6 == cudaSuccess; ++h)
        for (int m = 0; m < 3; ++m) {
          e6 = cudaMemcpy(c->ws + E.off_qkvh[l] + ((size_t)h * 192 + m * 64) * D * 2,
                          c->wptr<uint8_t>(p + "mha/Wqkv") + ((size_t)m * D + h * 64) * D * 2, (size_t)64 * D * 2,
                          cudaMemcpyDeviceToDevice);
          for (int j = 0; j < 64; ++j) bh[h * 192 + m * 64 + j] = bq[m * D + h * 64 + j];
        }
      if (e6 == cudaSuccess) e6 = cudaMemcpy(c->ws + E.off_bqkvh[l], bh.data(), 3 * D * 4, cudaMemcpyHostToDevice);
      if (e6 != cudaSuccess) return c->fail(CVR_E_CUDA, "assembling the head-major Wqkv");
      ok &= encode_tmap_bf16(&E.Wqkvh[l], c->ws + E.off_qkvh[l], 3 * D, D, D, 192, &er) == 0;
    }
  }
  if (!ok) return c->fail(CVR_E_CUDA, "tensor map encode: %s", er ? er : "?");
  // head MLP: same plan as the low-rank path (GemmPlan per mlp layer)
  c->plan.clear();
  int K = W;
  for (int i = 0; i < c->n_mlp; ++i) {
    const bool last = i + 1 == c->n_mlp;
    GemmPlan g;
    g.N = c->mlp[i];
    g.K = K;
    g.BN = last ? (c->head_parts ? 256 : c->mlp[i]) : pick_bn(c->mlp[i], c->max_batch);
    g.epi = last ? (c->head_parts ? EPI_HEAD_PARTIAL : EPI_HEAD) : EPI_BIAS_RELU;
    g.pair = c->pair_ens;
    if (encode_tmap_bf16(&g.tmB, c->wptr("mlp/" + std::to_string(i) + "/W"), g.N, K, K, g.pair ? g.BN / 2 : g.BN, &er) != 0)
      return c->fail(CVR_E_CUDA, "tensor map encode: %s", er ? er : "?");
    c->plan.push_back(g);
    K = c->mlp[i];
  }
  return CVR_OK;
}

// MaskNet plan: V_all / c_all assembled from the loaded blocks (block j = p * S + q), B maps of the
// projection, the hidden GEMM and every block's U; then the MLP tower as on the low-rank path.
int encode_plan_masknet(cvr_ctx* c) {
  const char* er = nullptr;
  auto& K = c->mk;
  const int S = c->n_cross, nb = K.P * S, r = c->r, Wp = K.Wp;
  for (int p = 0; p < K.P; ++p)
    for (int q = 0; q < S; ++q) {
      const int j = p * S + q;
      const std::string n = "mask/" + std::to_string(p) + "/" + std::to_string(q) + "/";
      cudaError_t e1 = cudaMemcpy(c->ws + K.off_Vall + (size_t)j * r * Wp * 2, c->wptr(n + "V"), (size_t)r * Wp * 2,
                                  cudaMemcpyDeviceToDevice);
      cudaError_t e2 = cudaMemcpy(c->ws + K.off_call + (size_t)j * r * 4, c->wptr(n + "c"), (size_t)r * 4,
                                  cudaMemcpyDeviceToDevice);
      if (e1 != cudaSuccess || e2 != cudaSuccess) return c->fail(CVR_E_CUDA, "assembling the MaskNet V_all / c_all");
      if (S == 1) {  // parallel-only: all branches' mask GEMMs run as one grouped launch
        cudaError_t e3 = cudaMemcpy(c->ws + K.off_Uall + (size_t)p * Wp * r * 2, c->wptr(n + "U"), (size_t)Wp * r * 2,
                                    cudaMemcpyDeviceToDevice);
        cudaError_t e4 = cudaMemcpy(c->ws + K.off_ball + (size_t)p * Wp * 4, c->wptr(n + "b"), (size_t)Wp * 4,
                                    cudaMemcpyDeviceToDevice);
        if (e3 != cudaSuccess || e4 != cudaSuccess) return c->fail(CVR_E_CUDA, "assembling the MaskNet U_all / b_all");
      }
    }
  const int64_t M = c->max_batch;
  K.bn_proj = pick_bn(Wp, M);
  K.bn_h = pick_bn(nb * r, M);
  K.bn_u = Wp % 128 == 0 ? 128 : 64;
  bool ok = true;
  c->plan.clear();
  GemmPlan gp;
  gp.N = Wp;
  gp.K = (int)c->x0_ld;
  gp.BN = K.bn_proj;
  gp.epi = EPI_BIAS_RELU;
  ok &= encode_tmap_bf16(&gp.tmB, c->wptr("proj/W"), Wp, c->x0_ld, c->x0_ld, gp.BN, &er) == 0;
  c->plan.push_back(gp);  // plan[0]: projection
  ok &= encode_tmap_bf16(&K.tmB_Vall, c->ws + K.off_Vall, (int64_t)nb * r, Wp, Wp, K.bn_h, &er) == 0;
  if (S == 1) {
    ok &= encode_tmap_bf16(&K.tmB_Uall, c->ws + K.off_Uall, (int64_t)K.P * Wp, r, r, K.bn_u, &er) == 0;
    ok &= encode_tmap_bf16(&K.tm_Hall, c->ws + K.off_H, M, (int64_t)nb * r, (int64_t)nb * r, 128, &er) == 0;
  }
  K.tmB_U.assign(nb, CUtensorMap{});
  for (int p = 0; p < K.P; ++p)
    for (int q = 0; q < S; ++q)
      ok &= encode_tmap_bf16(&K.tmB_U[p * S + q],
                             c->wptr("mask/" + std::to_string(p) + "/" + std::to_string(q) + "/U"), Wp, r, r, K.bn_u,
                             &er) == 0;
  int Kd = K.P * Wp;
  for (int i = 0; i < c->n_mlp; ++i) {
    const bool last = i + 1 == c->n_mlp;
    GemmPlan g;
    g.N = c->mlp[i];
    g.K = Kd;
    g.epi = last ? (c->head_parts ? EPI_HEAD_PARTIAL : EPI_HEAD) : EPI_BIAS_RELU;
    g.BN = last ? (c->head_parts ? 256 : c->mlp[i]) : pick_bn(c->mlp[i], M);
    ok &= encode_tmap_bf16(&g.tmB, c->wptr("mlp/" + std::to_string(i) + "/W"), g.N, Kd, Kd, g.BN, &er) == 0;
    c->plan.push_back(g);  // plan[1 + i]: MLP
    Kd = c->mlp[i];
  }
  if (!ok) return c->fail(CVR_E_CUDA, "tensor map encode: %s", er ? er : "?");
  return CVR_OK;
}

// widen a caller weight (fp32 / bf16) to host fp32
std::vector<float> fetch_f32(const void* d, int dtype, size_t n, cudaError_t& e) {
  std::vector<float> out(n);
  if (dtype == CVR_F32) {
    e = cudaMemcpy(out.data(), d, n * 4, cudaMemcpyDeviceToHost);
  } else {
    std::vector<uint16_t> tmp(n);
    e = cudaMemcpy(tmp.data(), d, n * 2, cudaMemcpyDeviceToHost);
    for (size_t i = 0; i < n; ++i) {
      uint32_t u = (uint32_t)tmp[i] << 16;
      float f;
      memcpy(&f, &u, 4);
      out[i] = f;
    }
  }
  return out;
}

}  // namespace

int cvr_load_weights(cvr_ctx* c, int n, const char* const* names, const void* const* ptrs, const int* dtypes,
                     const int* ndims, const int64_t* shapes) {
  if (!c || n < 0 || !names || !ptrs || !dtypes || !ndims || !shapes) return CVR_E_ARG;
  CVR_FORWARD_LANES(c, cvr_load_weights(lc_, n, names, ptrs, dtypes, ndims, shapes));
  if (!c->cuda_ready) return c->fail(CVR_E_STATE, "cvr_load_weights before cvr_set_workspace");
  std::vector<int> seen(c->wslots.size(), -1);
  int64_t so = 0;
  std::vector<int64_t> soff(n);
  for (int i = 0; i < n; ++i) {
    if (!names[i] || !ptrs[i] || ndims[i] < 1 || ndims[i] > 4) return c->fail(CVR_E_ARG, "weight entry %d malformed", i);
    soff[i] = so;
    so += ndims[i];
    int j = -1;
    for (size_t q = 0; q < c->wslots.size(); ++q)
      if (c->wslots[q].name == names[i]) j = (int)q;
    if (j < 0) return c->fail(CVR_E_SHAPE, "unexpected weight name '%s'", names[i]);
    if (seen[j] >= 0) return c->fail(CVR_E_SHAPE, "weight '%s' given twice", names[i]);
    seen[j] = i;
    std::vector<int64_t> got(shapes + soff[i], shapes + soff[i] + ndims[i]);
    if (got != c->wslots[j].shape)
      return c->fail(CVR_E_SHAPE, "weight '%s': expected shape %s, got %s", names[i], shape_str(c->wslots[j].shape).c_str(),
                     shape_str(got).c_str());
    if (dtypes[i] != c->wslots[j].dtype)
      return c->fail(CVR_E_DTYPE, "weight '%s': expected dtype %d, got %d", names[i], c->wslots[j].dtype, dtypes[i]);
  }
  for (size_t q = 0; q < c->wslots.size(); ++q)
    if (seen[q] < 0) return c->fail(CVR_E_SHAPE, "missing weight '%s' %s", c->wslots[q].name.c_str(), shape_str(c->wslots[q].shape).c_str());

  for (size_t q = 0; q < c->wslots.size(); ++q) {
    WSlot& s = c->wslots[q];
    const int i = seen[q];
    size_t ne = 1;
    for (auto v : s.shape) ne *= (size_t)v;
    cudaError_t e = cudaSuccess;
    std::vector<float> h = fetch_f32(ptrs[i], dtypes[i], ne, e);
    if (e != cudaSuccess) return c->cuda_fail(e, "cvr_load_weights fetch");
    const std::string& nm = s.name;
    auto ends = [&](const char* suf) { return nm.size() >= strlen(suf) && nm.compare(nm.size() - strlen(suf), strlen(suf), suf) == 0; };
    std::vector<uint8_t> pack(s.bytes, 0);
    float* pf = reinterpret_cast<float*>(pack.data());
    uint16_t* pb = reinterpret_cast<uint16_t*>(pack.data());
    auto bf = [](float f) {  // exact: the value is already bf16-representable (stored dtype)
      uint32_t u;
      memcpy(&u, &f, 4);
      return (uint16_t)(u >> 16);
    };
    if (nm == "head/b") c->head_b = h[0];
    if (nm == "norm/std") {
      for (size_t j = 0; j < ne; ++j) pf[j] = std::max(h[j], 1e-8f);
    } else if (s.shape.size() == 1 || nm.rfind("norm/", 0) == 0 || nm.rfind("head/", 0) == 0) {
      for (size_t j = 0; j < ne; ++j) pf[j] = h[j];  // fp32 copy (zero padding beyond ne)
    } else if (c->backbone == CVR_DCN_FULL) {       // transpose [out, in] -> [in, out]
      const int64_t O = s.shape[0], I = s.shape[1];
      for (int64_t o = 0; o < O; ++o)
        for (int64_t ii = 0; ii < I; ++ii) pf[ii * O + o] = h[o * I + ii];
    } else if ((c->backbone == CVR_MASKNET && nm == "proj/W") ||
               (c->backbone != CVR_MASKNET && (ends("/V") || nm == "mlp/0/W"))) {  // [out, W] -> [out, x0_ld]
      const int64_t O = s.shape[0], I = s.shape[1];
      for (int64_t o = 0; o < O; ++o)
        for (int64_t ii = 0; ii < I; ++ii) pb[o * c->x0_ld + ii] = bf(h[o * I + ii]);
    } else {  // U [W, r] (rows beyond W stay zero) and the other MLP weights: as is
      for (size_t j = 0; j < ne; ++j) pb[j] = bf(h[j]);
    }
    e = cudaMemcpy(c->ws + s.off, pack.data(), s.bytes, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return c->cuda_fail(e, "cvr_load_weights upload");
    s.loaded = true;
  }
  c->drop_graphs();  // captured graphs hold the old plan's tensor maps / head bias by value
  if (c->backbone == CVR_DCN_LOWRANK) {
    int st = encode_plan(c);
    if (st != CVR_OK) return st;
  } else if (c->backbone == CVR_ENSEMBLE) {
    int st = encode_plan_ensemble(c);
    if (st != CVR_OK) return st;
  } else if (c->backbone == CVR_MASKNET) {
    int st = encode_plan_masknet(c);
    if (st != CVR_OK) return st;
  }
  c->weights_loaded = true;
  return CVR_OK;
}

}  // extern "C"

namespace {

int check_ready(cvr_ctx* c, bool need_tables, bool need_weights) {
  if (!c->cuda_ready) return c->fail(CVR_E_STATE, "workspace not set");
  if (need_tables && !c->tables_loaded) return c->fail(CVR_E_STATE, "tables not loaded");
  if (need_weights && !c->weights_loaded) return c->fail(CVR_E_STATE, "weights not loaded");
  return CVR_OK;
}

EmbedArgs embed_args(cvr_ctx* c, const int32_t* idx, const int32_t* off, int64_t nnz, int B, const float* dense,
                     void* out, int64_t out_ld, void* x0, int Bd) {
  EmbedArgs a{};
  a.tables = c->at<TableDesc>(c->off_tables);
  a.indices = idx;
  a.offsets = off;
  a.nnz = nnz;
  a.B = B;
  a.T = (int)c->local_tables.size();
  a.d = c->d;
  a.emb_dtype = c->emb_dtype;
  a.out_dtype = c->act;
  a.out = out;
  a.out_ld = out_ld;
  a.out_tstride = c->d;
  a.dense = dense;
  a.Bd = Bd;
  a.F = c->F;
  a.mean = c->F ? c->wptr<float>("norm/mean") : nullptr;
  a.sigma = c->F ? c->wptr<float>("norm/std") : nullptr;
  a.x0 = x0;
  a.x0_ld = c->x0_ld;
  a.dense_col0 = (int64_t)c->T * c->d;
  a.pad_col0 = c->W;
  a.pad_col1 = c->x0_ld;
  a.flag = c->at<int>(c->off_flag);
  a.call = c->call;
  return a;
}

// S2 + S3.  Executor stages (c->call set): B is max_batch (grid size); the kernel reads the batch from the block.
int do_embed(cvr_ctx* c, const int32_t* idx, const int32_t* off, int64_t nnz, int B, const float* dense, void* x0,
             cudaStream_t s, int blocks_per_sm = 0, const uint64_t* keys = nullptr) {
  if (c->F && !c->slot("norm/mean")->loaded) return c->fail(CVR_E_STATE, "norm/mean,std not loaded");
  EmbedArgs a = embed_args(c, idx, off, nnz, B, dense, x0, c->x0_ld, x0, B);
  a.keys = keys;
  a.blocks_per_sm = blocks_per_sm;
  c->pbeg(s);
  cudaError_t e = launch_embed(a, c->num_sms, s);
  c->pend(K_EMBED, s);
  if (e != cudaSuccess) return c->cuda_fail(e, "embed launch");
  return CVR_OK;
}

// M: rows of the A operand (examples, or tokens = examples x m_mult); executor stages pass max_batch x m_mult
GemmArgs gemm_args(cvr_ctx* c, const GemmPlan& g, const CUtensorMap* A, int M, int m_mult = 1) {
  GemmArgs a{};
  a.tmA = A;
  a.tmB = &g.tmB;
  a.M = M;
  a.N = g.N;
  a.K = g.K;
  a.BN = g.BN;
  a.epi = g.epi;
  a.num_sms = c->num_sms;
  a.pdl = c->pdl;
  a.cta_pair = g.pair;
  a.no_prefetch_b = !c->prefetch_b;
  a.call = c->call;
  a.m_mult = m_mult;
  {  // several tiles per CTA: the epilogue overlaps the next mainloop, keep the CTA small (Cfg::EPW)
    const int rows = g.pair ? 256 : 128, units = g.pair ? c->num_sms / 2 : c->num_sms;
    const int64_t tiles = (int64_t)((M + rows - 1) / rows) * (g.N / g.BN);
    a.epw1 = c->epw_mode == 0 || (c->epw_mode == 2 && tiles > 2 * units);
  }
  if (c->gdbg && c->gdbg_n < 32) a.dbg = c->gdbg + (size_t)(c->gdbg_n++) * 160 * 8;
  return a;
}

cudaError_t run_gemm(cvr_ctx* c, const GemmArgs& a, int kid, cudaStream_t s) {
  if (c->only_kid >= 0) {  // cvr_repeat_kernel: this role only, back to back (programmatic launches)
    if (kid != c->only_kid) return cudaSuccess;
    for (int i = 0; i < c->only_reps; ++i) {
      cudaError_t r = launch_gemm_bf16(a, s);
      ++c->launches;
      if (r != cudaSuccess) return r;
    }
    return cudaSuccess;
  }
  if (a.dbg) c->gdbg_kid.push_back(kid);
  c->pbeg(s);
  cudaError_t r = launch_gemm_bf16(a, s);
  c->pend(kid, s);
  return r;
}

// S6 + S7: hidden MLP layers (bias + ReLU) then the head: fused into the last GEMM's epilogue when
// the last width fits one N tile (<= 256), else 256-wide partial dot products + a fixed-order finaliser.
int run_mlp_head(cvr_ctx* c, const CUtensorMap* tm_in, size_t pi, int B, float* scores, cudaStream_t s) {
  cudaError_t e;
  for (int i = 0; i < c->n_mlp; ++i) {
    const GemmPlan& g = c->plan[pi++];
    GemmArgs a = gemm_args(c, g, tm_in, B);
    a.bias = c->wptr<float>("mlp/" + std::to_string(i) + "/b");
    int kid = K_GEMM_MLP;
    if (g.epi == EPI_HEAD) {
      a.head_w = c->wptr<float>("head/w");
      a.head_b = c->head_b;
      a.scores = scores;
      kid = K_GEMM_HEAD;
    } else if (g.epi == EPI_HEAD_PARTIAL) {
      a.head_w = c->wptr<float>("head/w");
      a.partial = c->at<float>(c->off_hpart);
      kid = K_GEMM_HEAD;
    } else {
      a.tmOut = &c->st_h[i];
    }
    if ((e = run_gemm(c, a, kid, s)) != cudaSuccess) return c->cuda_fail(e, "gemm MLP launch");
    if (g.epi == EPI_HEAD_PARTIAL && c->only_kid < 0) {
      c->pbeg(s);
      e = launch_head_finalize(c->at<float>(c->off_hpart), c->head_parts, c->head_b, scores, B, s, c->call);
      c->pend(K_HEAD_FIN, s);
      if (e != cudaSuccess) return c->cuda_fail(e, "head finalize launch");
    }
    if (g.epi == EPI_BIAS_RELU) tm_in = &c->tm_h[i];
  }
  return CVR_OK;
}

// S5' (config 4, A20/A26): per layer Y = LN_token(DCN(X) + MHA(X) + FFN(X)); the branch sum is kept in
// fp32 (S) and the LN runs in the FFN2 epilogue.
int do_dense_ensemble(cvr_ctx* c, const CUtensorMap* flat_x0, const CUtensorMap* tok_x0, int B, float* scores,
                      cudaStream_t s) {
  auto& E = c->ens;
  cudaError_t e;
  const int D = c->d, W = (int)c->x0_ld, r = c->r, T = c->T, BT = B * T;
  float* S = c->at<float>(E.off_S);
  const CUtensorMap* flat_xl = flat_x0;
  const CUtensorMap* tok_xl = tok_x0;
  // M rows: B (flat [B, W] operands) or BT (token [B*T, D] operands, m_mult = T)
  auto ga = [&](const CUtensorMap* A, const CUtensorMap* Bm, int M, int N, int K, int BN, Epi epi) {
    GemmArgs a{};
    a.tmA = A;
    a.tmB = Bm;
    a.no_prefetch_b = !c->prefetch_b;
    a.M = M;
    a.N = N;
    a.K = K;
    a.BN = BN;
    a.epi = epi;
    a.num_sms = c->num_sms;
    a.pdl = c->pdl;
    a.cta_pair = c->pair_ens;
    a.call = c->call;
    a.m_mult = M == BT ? T : 1;
    const int rows = c->pair_ens ? 256 : 128, units = c->pair_ens ? c->num_sms / 2 : c->num_sms;
    const int64_t tiles = (int64_t)((M + rows - 1) / rows) * (N / BN);
    a.epw1 = c->epw_mode == 0 || (c->epw_mode == 2 && tiles > 2 * units);
    if (c->gdbg && c->gdbg_n < 32) a.dbg = c->gdbg + (size_t)(c->gdbg_n++) * 160 * 8;  // CVR_GEMM_TIMELINE
    return a;
  };
  for (int l = 0; l < c->n_cross; ++l) {
    const std::string p = "ens/" + std::to_string(l) + "/";
    const bool even = l % 2 == 0;
    // DCN branch: t = X V^T ; S = x0 * (t U^T + b) + X   (fp32, A26)
    GemmArgs a1 = ga(flat_xl, &E.V[l], B, r, W, 128, EPI_STORE);
    // t = X V^T has only (B / 128) x (r / 128) tiles of a very long K (W = 16384): 2-CTA 256 x 128 tiles give
    // 1.73 waves (the second wave 73% full: measured 164 us, every CTA's tile ~82 us); 128 x 256 single-CTA tiles
    // fit one wave when (B / 128) (r / 256) <= #SMs
    if (c->ens_xv_wave && r % 256 == 0 && (int64_t)((B + 127) / 128) * (r / 256) <= c->num_sms) {
      a1.BN = 256;
      a1.cta_pair = false;
      a1.tmB = &E.V256[l];
      a1.epw1 = false;
    }
    a1.tmOut = &c->st_t;
    if ((e = run_gemm(c, a1, K_GEMM_V, s)) != cudaSuccess) return c->cuda_fail(e, "ens V");
    GemmArgs a2 = ga(&c->tm_t, &E.U[l], B, W, r, c->ens_u_bn, EPI_CROSS_F32);
    a2.tmX0 = flat_x0;
    a2.tmXl = flat_xl;
    a2.bias = c->wptr<float>(p + "dcn/b");
    a2.out_f32 = S;
    a2.ld_f32 = W;
    if (c->f32_tma_store && E.st_S_ok) a2.tmOut = &E.st_S;  // staged, coalesced TMA stores of S
    if ((e = run_gemm(c, a2, K_GEMM_U, s)) != cudaSuccess) return c->cuda_fail(e, "ens U");
    // MHA branch: qkv = X Wqkv^T + b ; O = attention ; S += O Wo^T + bo
    __nv_bfloat16* cat = c->at<__nv_bfloat16>(E.off_cat);
    if (c->ens_fused_attn && D == 64 * c->n_heads) {
      // one GEMM: each 128-token x 192 tile [q_h | k_h | v_h] (+ b) is attended in its epilogue, O -> cat[:, 64 h ..]
      // (the qkv tensor never reaches HBM; same bf16 roundings and attention core as qkv GEMM + mha64)
      GemmArgs a3 = ga(tok_xl, &E.Wqkvh[l], BT, 3 * D, D, 192, c->ens_attn_tc ? EPI_ATTN_TC : EPI_ATTN);
      a3.cta_pair = false;
      a3.bias = c->at<float>(E.off_bqkvh[l]);
      a3.out_bf16 = cat;
      a3.ld_x = D + c->ffn;
      if (c->ens_attn_tc) a3.tmOut = &E.tm_cat;  // O: 128 x 64 boxes at cat[m0.., 64 h] (TMA store)
      if ((e = run_gemm(c, a3, K_ENS_QKV_ATTN, s)) != cudaSuccess) return c->cuda_fail(e, "ens qkv + attention");
    } else {
      GemmArgs a3 = ga(tok_xl, &E.Wqkv[l], BT, 3 * D, D, 256, EPI_BIAS);
      a3.tmOut = &E.st_qkv;
      a3.bias = c->wptr<float>(p + "mha/bqkv");
      if ((e = run_gemm(c, a3, K_ENS_QKV, s)) != cudaSuccess) return c->cuda_fail(e, "ens qkv");
      if (c->only_kid < 0) c->pbeg(s);
      if (c->only_kid < 0) {
        e = launch_mha64(c->at<__nv_bfloat16>(E.off_qkv), cat, D + c->ffn, B, c->n_heads, s, c->call);  // O -> cat[:, :D]
        c->pend(K_MHA, s);
        if (e != cudaSuccess) return c->cuda_fail(e, "mha64");
      }
    }
    if (c->ens_ffn_fused && D == 256 && c->ffn % 128 == 0) {
      // FFN1 + out-projection + FFN2 + branch-sum LN in one kernel: h stays in TMEM / shared memory
      FfnArgs f{};
      f.tmX = tok_xl;
      f.tmO = &E.tm_cat;
      f.tmW1 = &E.W1f[l];
      f.tmW2 = &E.W2f[l];
      f.tmWo = &E.Wof[l];
      f.tmS = &E.ld_Stok;
      f.tmOut = even ? &E.sttok_xa : &E.sttok_xb;
      f.b1 = c->wptr<float>(p + "ffn/b1");
      f.bcat = c->at<float>(E.off_catb[l]);
      f.gamma = c->wptr<float>(p + "ln/gamma");
      f.beta = c->wptr<float>(p + "ln/beta");
      f.M = BT;
      f.F = c->ffn;
      f.D = D;
      f.m_mult = T;
      f.num_sms = c->num_sms;
      f.pdl = c->pdl;
      f.call = c->call;
      if (c->only_kid < 0 || c->only_kid == K_ENS_FFN_FUSED) {
        const int reps = c->only_kid == K_ENS_FFN_FUSED ? c->only_reps : 1;
        for (int i = 0; i < reps; ++i) {
          c->pbeg(s);
          e = launch_ffn_fused(f, s);
          c->pend(K_ENS_FFN_FUSED, s);
          if (e != cudaSuccess) return c->cuda_fail(e, "ens fused ffn");
        }
      }
      flat_xl = even ? &E.flat_xa : &E.flat_xb;
      tok_xl = even ? &E.tok_xa : &E.tok_xb;
      continue;
    }
    // FFN hidden -> cat[:, D:]
    GemmArgs a5 = ga(tok_xl, &E.W1[l], BT, c->ffn, D, 256, EPI_BIAS_RELU);
    a5.tmOut = &E.st_hf;
    a5.bias = c->wptr<float>(p + "ffn/b1");
    if ((e = run_gemm(c, a5, K_ENS_FFN1, s)) != cudaSuccess) return c->cuda_fail(e, "ens ffn1");
    // X' = LN([O | h] [Wo | W2]^T + (bo + b2) + S) * gamma + beta   (S = DCN branch, fp32)
    GemmArgs a6 = ga(&E.tm_cat, &E.Wcat[l], BT, D, D + c->ffn, 256, EPI_SUM_LN);
    a6.tmOut = even ? &E.sttok_xa : &E.sttok_xb;
    a6.bias = c->at<float>(E.off_catb[l]);
    a6.in_f32 = S;
    a6.ld_in = D;
    a6.tmX0 = &E.ld_Stok;  // S chunks by TMA (EPI_SUM_LN's input ring)
    a6.gamma = c->wptr<float>(p + "ln/gamma");
    a6.beta = c->wptr<float>(p + "ln/beta");
    if ((e = run_gemm(c, a6, K_ENS_FFN2_LN, s)) != cudaSuccess) return c->cuda_fail(e, "ens out-proj+ffn2+ln");
    flat_xl = even ? &E.flat_xa : &E.flat_xb;
    tok_xl = even ? &E.tok_xa : &E.tok_xb;
  }
  return run_mlp_head(c, flat_xl, 0, B, scores, s);
}

// MaskNet dense stage: projection, all blocks' mask hiddens in one GEMM, one mask GEMM
// per block (EPI_MASK: (H U^T + b) * x), then the MLP tower + head on the concatenated branches.
int do_dense_masknet(cvr_ctx* c, const CUtensorMap* tm_x0, int B, float* scores, cudaStream_t s) {
  auto& K = c->mk;
  const int S = c->n_cross, nb = K.P * S;
  cudaError_t e;
  GemmArgs a = gemm_args(c, c->plan[0], tm_x0, B);  // x0' = ReLU(x0 W_in^T + b_in)
  a.bias = c->wptr<float>("proj/b");
  a.tmOut = &K.st_x0p;
  if ((e = run_gemm(c, a, K_MASK_PROJ, s)) != cudaSuccess) return c->cuda_fail(e, "MaskNet projection");
  GemmPlan gh;
  gh.N = nb * c->r;
  gh.K = K.Wp;
  gh.BN = K.bn_h;
  gh.epi = EPI_BIAS_RELU;
  GemmArgs ah = gemm_args(c, gh, &K.tm_x0p, B);  // H = ReLU(x0' V_all^T + c_all)
  ah.tmB = &K.tmB_Vall;
  ah.bias = c->at<float>(K.off_call);
  ah.tmOut = &K.st_H;
  if ((e = run_gemm(c, ah, K_MASK_HIDDEN, s)) != cudaSuccess) return c->cuda_fail(e, "MaskNet mask hidden");
  if (S == 1 && c->mask_grouped) {
    // every branch's block in ONE grouped launch: N = P * W' over cat, branch g = n / W' reads H columns
    // [g r, (g + 1) r), U rows of branch g (stacked), bias b_g, and x0' columns n - g W'
    GemmPlan gu;
    gu.N = K.P * K.Wp;
    gu.K = c->r;
    gu.BN = K.bn_u;
    gu.epi = EPI_MASK;
    GemmArgs au = gemm_args(c, gu, &K.tm_Hall, B);
    au.tmB = &K.tmB_Uall;
    au.tmXl = &K.tm_x0p;
    au.bias = c->at<float>(K.off_ball);
    au.tmOut = &K.tm_cat_st;
    au.group_n = K.Wp;
    if ((e = run_gemm(c, au, K_MASK_MUL, s)) != cudaSuccess) return c->cuda_fail(e, "MaskNet grouped mask blocks");
  } else {
    for (int p = 0; p < K.P; ++p) {
      const CUtensorMap* x_in = &K.tm_x0p;
      for (int q = 0; q < S; ++q) {
        const int j = p * S + q;
        GemmPlan gu;
        gu.N = K.Wp;
        gu.K = c->r;
        gu.BN = K.bn_u;
        gu.epi = EPI_MASK;
        GemmArgs au = gemm_args(c, gu, &K.tm_Hblk[j], B);
        au.tmB = &K.tmB_U[j];
        au.tmXl = x_in;
        au.bias = c->wptr<float>("mask/" + std::to_string(p) + "/" + std::to_string(q) + "/b");
        au.tmOut = q + 1 == S ? &K.st_cat[p] : &K.st_tmp[q % 2];
        if ((e = run_gemm(c, au, K_MASK_MUL, s)) != cudaSuccess) return c->cuda_fail(e, "MaskNet mask block");
        x_in = &K.tm_tmp[q % 2];
      }
    }
  }
  // MLP tower + head on cat [B, P * Wp]: plan[1..]
  return run_mlp_head(c, &K.tm_cat, 1, B, scores, s);
}

int do_dense(cvr_ctx* c, const void* x0, const CUtensorMap* tm_x0, const CUtensorMap* tm_x0_tok, int B, float* scores,
             cudaStream_t s) {
  c->gdbg_n = 0;  // CVR_GEMM_TIMELINE: stamps of this stage's GEMMs start at slot 0
  c->gdbg_kid.clear();
  cudaError_t e = cudaSuccess;
  if (c->backbone == CVR_DCN_FULL) {
    DenseF32Args a{};
    a.x0 = reinterpret_cast<const float*>(x0);
    a.x0_ld = c->x0_ld;
    a.B = B;
    a.W = c->W;
    a.n_cross = c->n_cross;
    for (int l = 0; l < c->n_cross; ++l) {
      a.WT[l] = c->wptr<float>("dcn/" + std::to_string(l) + "/W");
      a.bias[l] = c->wptr<float>("dcn/" + std::to_string(l) + "/b");
    }
    a.n_mlp = c->n_mlp;
    a.dims[0] = c->W;
    for (int i = 0; i < c->n_mlp; ++i) {
      a.dims[i + 1] = c->mlp[i];
      a.MT[i] = c->wptr<float>("mlp/" + std::to_string(i) + "/W");
      a.mb[i] = c->wptr<float>("mlp/" + std::to_string(i) + "/b");
    }
    a.head_w = c->wptr<float>("head/w");
    a.head_b = c->wptr<float>("head/b");
    a.scores = scores;
    a.call = c->call;
    c->pbeg(s);
    e = launch_dense_f32(a, s);
    c->pend(K_DENSE_F32, s);
    if (e != cudaSuccess) return c->cuda_fail(e, "dense_f32 launch");
    return CVR_OK;
  }
  if (c->backbone == CVR_ENSEMBLE) return do_dense_ensemble(c, tm_x0, tm_x0_tok, B, scores, s);
  if (c->backbone == CVR_MASKNET) return do_dense_masknet(c, tm_x0, B, scores, s);
  // ---- bf16 low-rank DCN-v2 on tcgen05: per layer t = x_l V^T (EPI_STORE), x_{l+1} = x0 * (t U^T + b) + x_l
  const CUtensorMap* tm_xl = tm_x0;
  size_t pi = 0;
  for (int l = 0; l < c->n_cross; ++l) {
    const GemmPlan& gv = c->plan[pi++];
    const GemmPlan& gu = c->plan[pi++];
    const bool even = l % 2 == 0;
    GemmArgs av = gemm_args(c, gv, tm_xl, B);
    av.tmOut = &c->st_t;
    if ((e = run_gemm(c, av, K_GEMM_V, s)) != cudaSuccess) return c->cuda_fail(e, "gemm V launch");
    GemmArgs au = gemm_args(c, gu, &c->tm_t, B);
    au.tmOut = even ? &c->st_xa : &c->st_xb;
    au.tmX0 = tm_x0;
    au.tmXl = tm_xl;
    au.bias = c->wptr<float>("dcn/" + std::to_string(l) + "/b");
    if ((e = run_gemm(c, au, K_GEMM_U, s)) != cudaSuccess) return c->cuda_fail(e, "gemm U launch");
    tm_xl = even ? &c->tm_xa : &c->tm_xb;
  }
  return run_mlp_head(c, tm_xl, pi, B, scores, s);
}

// x0 tensor maps of a caller buffer (standalone cvr_dense on a buffer that is not an x0 slot)
int user_x0_maps(cvr_ctx* c, const void* d_x0, int batch, CUtensorMap* tm, CUtensorMap* tmt) {
  const char* er = nullptr;
  if (encode_tmap_bf16(tm, d_x0, batch, c->x0_ld, c->x0_ld, 128, &er) != 0 ||
      (c->backbone == CVR_ENSEMBLE && encode_tmap_bf16(tmt, d_x0, (int64_t)batch * c->T, c->d, c->d, 128, &er) != 0))
    return c->fail(CVR_E_CUDA, "tensor map encode: %s", er ? er : "?");
  return CVR_OK;
}

// Run one executor stage for slot `slot`: replay its graph (captured at first use; the batch is read from the
// per-call block, so the same graph serves every batch and batch size), or launch directly (graphs off, while
// profiling, or inside a caller's own capture).
template <typename F>
int run_stage(cvr_ctx* c, int kind, int slot, int bucket, cudaStream_t s, F&& enqueue, bool launch = true) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (!c->use_graphs || s == nullptr || c->prof_on || cudaStreamIsCapturing(s, &cs) != cudaSuccess ||
      cs != cudaStreamCaptureStatusNone)
    return launch ? enqueue(s) : CVR_OK;
  cudaGraphExec_t& ge = c->gexec[kind][slot][bucket];
  if (!ge) {
    const int64_t l0 = c->launches;
    cudaError_t e = cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    if (e != cudaSuccess) return c->cuda_fail(e, "cudaStreamBeginCapture");
    int st = enqueue(s);
    cudaGraph_t graph = nullptr;
    e = cudaStreamEndCapture(s, &graph);
    const int64_t nk = c->launches - l0;
    c->launches = l0;
    if (st != CVR_OK) {
      if (graph) cudaGraphDestroy(graph);
      return st;
    }
    if (e != cudaSuccess) return c->cuda_fail(e, "cudaStreamEndCapture");
    e = cudaGraphInstantiate(&ge, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) {
      ge = nullptr;
      return c->cuda_fail(e, "cudaGraphInstantiate");
    }
    c->gkernels[kind][slot][bucket] = nk;
    ++c->graph_captures;
  }
  if (!launch) return CVR_OK;  // (capture only: cvr_warm_graphs)
  cudaError_t e = cudaGraphLaunch(ge, s);
  if (e != cudaSuccess) return c->cuda_fail(e, "cudaGraphLaunch");
  c->launches += c->gkernels[kind][slot][bucket];
  return CVR_OK;
}

}  // namespace

extern "C" {

int cvr_embed(cvr_ctx* c, const int32_t* d_indices, const int32_t* d_offsets, int64_t nnz, int batch,
              const float* d_dense, void* d_x0, cvr_stream_t stream) {
  if (!c) return CVR_E_ARG;
  int st = check_ready(c, true, false);
  if (st) return st;
  if (c->world != 1) return c->fail(CVR_E_STATE, "cvr_embed is unsharded; use cvr_embed_shard");
  if (batch < 0 || batch > c->max_batch) return c->fail(CVR_E_ARG, "batch %d outside [0, %d]", batch, c->max_batch);
  if (!d_offsets || !d_x0 || (nnz > 0 && !d_indices) || (c->F && batch && !d_dense) || nnz < 0)
    return c->fail(CVR_E_ARG, "null pointer or negative nnz");
  return do_embed(c, d_indices, d_offsets, nnz, batch, d_dense, d_x0, (cudaStream_t)stream);
}

int cvr_set_feature_spec(cvr_ctx* c, int n, const int64_t* vocab, const int* pool_mode) {
  if (!c || !vocab || !pool_mode) return CVR_E_ARG;
  CVR_FORWARD_LANES(c, cvr_set_feature_spec(lc_, n, vocab, pool_mode));
  if (n != c->T) return c->fail(CVR_E_SHAPE, "feature spec: expected %d tables, got %d", c->T, n);
  for (int t = 0; t < n; ++t) {
    if (pool_mode[t] != 0 && pool_mode[t] != 1) return c->fail(CVR_E_ARG, "table %d: pool_mode must be 0 (sum) or 1 (mean)", t);
    if (vocab[t] < 0 || (vocab[t] > 0 && vocab[t] + 1 > c->rows[t]))
      return c->fail(CVR_E_SHAPE, "table %d: vocab %lld needs rows >= vocab + 1 (the unseen row), table has %lld", t,
                     (long long)vocab[t], (long long)c->rows[t]);
  }
  c->any_mean = false;
  for (int t = 0; t < n; ++t) {
    c->tvocab[t] = vocab[t];
    c->tmean[t] = pool_mode[t];
    c->any_mean |= pool_mode[t] == 1;
  }
  if (c->tables_loaded) {
    for (size_t i = 0; i < c->local_tables.size(); ++i) {
      c->htables[i].vocab = c->tvocab[c->local_tables[i]];
      c->htables[i].magic = c->htables[i].vocab > 0 ? ~0ull / (uint64_t)c->htables[i].vocab : 0ull;
      c->htables[i].mean = c->tmean[c->local_tables[i]];
    }
    cudaError_t e = cudaMemcpy(c->ws + c->off_tables, c->htables.data(), sizeof(TableDesc) * c->htables.size(),
                               cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return c->cuda_fail(e, "cvr_set_feature_spec");
  }
  return CVR_OK;
}

int cvr_embed_keys(cvr_ctx* c, const uint64_t* d_keys, const int32_t* d_offsets, int64_t nnz, int batch,
                   const float* d_dense, void* d_x0, cvr_stream_t stream) {
  if (!c) return CVR_E_ARG;
  int st = check_ready(c, true, false);
  if (st) return st;
  if (c->world != 1) return c->fail(CVR_E_STATE, "cvr_embed_keys is unsharded");
  for (int t = 0; t < c->T; ++t)
    if (c->tvocab[t] <= 0) return c->fail(CVR_E_STATE, "table %d has no hash vocab (cvr_set_feature_spec)", t);
  if (batch < 0 || batch > c->max_batch) return c->fail(CVR_E_ARG, "batch %d outside [0, %d]", batch, c->max_batch);
  if (!d_offsets || !d_x0 || (nnz > 0 && !d_keys) || (c->F && batch && !d_dense) || nnz < 0)
    return c->fail(CVR_E_ARG, "null pointer or negative nnz");
  return do_embed(c, nullptr, d_offsets, nnz, batch, d_dense, d_x0, (cudaStream_t)stream, 0, d_keys);
}

int cvr_dense(cvr_ctx* c, const void* d_x0, int batch, float* d_scores, cvr_stream_t stream) {
  if (!c) return CVR_E_ARG;
  int st = check_ready(c, false, true);
  if (st) return st;
  if (batch < 0 || batch > c->max_batch) return c->fail(CVR_E_ARG, "batch %d outside [0, %d]", batch, c->max_batch);
  if (!d_x0 || !d_scores) return c->fail(CVR_E_ARG, "null pointer");
  if (batch == 0) return CVR_OK;
  const CUtensorMap* tm = nullptr;
  const CUtensorMap* tmt = nullptr;
  CUtensorMap um, umt;
  if (c->backbone != CVR_DCN_FULL) {
    const bool ens = c->backbone == CVR_ENSEMBLE;
    int slot = -1;
    for (int i = 0; i < cvr_ctx::kSlots; ++i)
      if (d_x0 == c->ws + c->off_x0[i]) slot = i;
    if (slot >= 0) {
      tm = ens ? &c->ens.flat_x0[slot] : &c->tm_x0slot[slot];
      tmt = &c->ens.tok_x0[slot];
    } else {
      if ((st = user_x0_maps(c, d_x0, batch, &um, &umt)) != CVR_OK) return st;
      tm = &um;
      tmt = &umt;
    }
  }
  return do_dense(c, d_x0, tm, tmt, batch, d_scores, (cudaStream_t)stream);
}

}  // extern "C"

namespace {
// the two-stream executor behind cvr_score (row ids) and cvr_score_keys (raw keys, hashed in the gather):
// slot = k % kSlots; on s_embed: [wait dense(k-kSlots)] -> set_call(slot) -> embed graph(slot) -> event; on s_dense:
// [wait embed(k)] -> dense graph(slot) -> event.  Both graphs read the batch from the slot's call block.
int score_impl(cvr_ctx* c, const int32_t* d_indices, const uint64_t* d_keys, const int32_t* d_offsets, int64_t nnz,
               int batch, const float* d_dense, float* d_scores, cvr_stream_t s_embed, cvr_stream_t s_dense,
               cudaStream_t s_after_wait = nullptr) {
  if (!c) return CVR_E_ARG;
  int st = check_ready(c, true, true);
  if (st) return st;
  if (c->world != 1) return c->fail(CVR_E_STATE, "cvr_score is unsharded");
  if (batch < 0 || batch > c->max_batch) return c->fail(CVR_E_ARG, "batch %d outside [0, %d]", batch, c->max_batch);
  if (!d_offsets || !d_scores || (nnz > 0 && !d_indices && !d_keys) || (c->F && batch && !d_dense) || nnz < 0)
    return c->fail(CVR_E_ARG, "null pointer or negative nnz");
  cudaStream_t se = (cudaStream_t)s_embed, sd = (cudaStream_t)s_dense;
  const int slot = (int)(c->k % cvr_ctx::kSlots);
  cudaError_t e = cudaSuccess;
  if (c->k >= cvr_ctx::kSlots) e = cudaStreamWaitEvent(se, c->ev_dense[slot], 0);  // dense(k-kSlots) released the slot
  if (e != cudaSuccess) return c->cuda_fail(e, "wait dense(k-kSlots)");
  CallArgs v{};
  v.indices = d_indices;
  v.keys = d_keys;
  v.offsets = d_offsets;
  v.dense = d_dense;
  v.scores = d_scores;
  v.nnz = nnz;
  v.B = batch;
  CallArgs* blk = c->at<CallArgs>(c->off_call[slot]);
  c->pbeg(se);
  e = launch_set_call(v, blk, se);
  c->pend(K_SET_CALL, se);
  if (e != cudaSuccess) return c->cuda_fail(e, "set_call launch");
  if (s_after_wait && (e = cudaStreamWaitEvent(se, c->ev_copy[slot], 0)) != cudaSuccess)  // host-fed: H2D landed
    return c->cuda_fail(e, "wait copy");
  void* x0 = c->ws + c->off_x0[slot];
  int bucket = 0;
  const int Bmax = c->bucket_rows(batch, &bucket);  // grid sizing only: the kernels read `batch` from the block
  c->call = blk;
  st = run_stage(c, d_keys ? cvr_ctx::G_EMBED_KEYS : cvr_ctx::G_EMBED, slot, bucket, se, [&](cudaStream_t s) {
    return do_embed(c, d_indices, d_offsets, nnz, Bmax, d_dense, x0, s, c->embed_bps_pipe, d_keys);
  });
  if (st) {
    c->call = nullptr;
    return st;
  }
  if ((e = cudaEventRecord(c->ev_embed[slot], se)) != cudaSuccess) st = c->cuda_fail(e, "record embed");
  if (!st && (e = cudaStreamWaitEvent(sd, c->ev_embed[slot], 0)) != cudaSuccess) st = c->cuda_fail(e, "wait embed");
  if (!st && batch > 0) {
    const bool ens = c->backbone == CVR_ENSEMBLE;
    const CUtensorMap* tm = (c->backbone == CVR_DCN_LOWRANK || c->backbone == CVR_MASKNET) ? &c->tm_x0slot[slot]
                            : ens ? &c->ens.flat_x0[slot] : nullptr;
    const CUtensorMap* tmt = ens ? &c->ens.tok_x0[slot] : nullptr;
    st = run_stage(c, cvr_ctx::G_DENSE, slot, bucket, sd,
                   [&](cudaStream_t s) { return do_dense(c, x0, tm, tmt, Bmax, d_scores, s); });
  }
  c->call = nullptr;
  if (st) return st;
  if ((e = cudaEventRecord(c->ev_dense[slot], sd)) != cudaSuccess) return c->cuda_fail(e, "record dense");
  c->k++;
  return CVR_OK;
}

// executor lanes: the library's stream pair of every lane, created at first use with the caller's priorities
int ensure_lane_streams(cvr_ctx* c, cudaStream_t s_embed, cudaStream_t s_dense) {
  if (c->lane_se[0]) return CVR_OK;
  int pe = 0, pd = 0;
  cudaError_t e = cudaStreamGetPriority(s_embed, &pe);
  if (e == cudaSuccess) e = cudaStreamGetPriority(s_dense, &pd);
  for (int i = 0; i < c->lanes && e == cudaSuccess; ++i) {
    e = cudaStreamCreateWithPriority(&c->lane_se[i], cudaStreamNonBlocking, pe);
    if (e == cudaSuccess) e = cudaStreamCreateWithPriority(&c->lane_sd[i], cudaStreamNonBlocking, pd);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->lane_in[i], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->lane_out[i], cudaEventDisableTiming);
  }
  if (e == cudaSuccess) return CVR_OK;
  for (int i = 0; i < cvr_ctx::kMaxLanes; ++i) {  // all or nothing: the next call retries from scratch
    if (c->lane_se[i]) cudaStreamDestroy(c->lane_se[i]);
    if (c->lane_sd[i]) cudaStreamDestroy(c->lane_sd[i]);
    if (c->lane_in[i]) cudaEventDestroy(c->lane_in[i]);
    if (c->lane_out[i]) cudaEventDestroy(c->lane_out[i]);
    c->lane_se[i] = c->lane_sd[i] = nullptr;
    c->lane_in[i] = c->lane_out[i] = nullptr;
  }
  return c->cuda_fail(e, "lane streams");
}

// call lane_k % lanes: its work waits for the caller's s_embed, runs on the lane's streams, and the caller's s_dense
// waits for its end
template <class F>
int lane_dispatch(cvr_ctx* c, cvr_stream_t s_embed, cvr_stream_t s_dense, F&& fn) {
  int st = ensure_lane_streams(c, (cudaStream_t)s_embed, (cudaStream_t)s_dense);
  if (st) return st;
  const int i = (int)(c->lane_k % c->lanes);
  cvr_ctx* t = c->lane(i);
  cudaError_t e = cudaEventRecord(c->lane_in[i], (cudaStream_t)s_embed);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(c->lane_se[i], c->lane_in[i], 0);
  if (e != cudaSuccess) return c->cuda_fail(e, "lane input order");
  st = fn(t, c->lane_se[i], c->lane_sd[i]);
  if (st) return i ? c->fail(st, "lane %d: %s", i, t->err.c_str()) : st;
  e = cudaEventRecord(c->lane_out[i], c->lane_sd[i]);
  if (e == cudaSuccess) e = cudaStreamWaitEvent((cudaStream_t)s_dense, c->lane_out[i], 0);
  if (e != cudaSuccess) return c->cuda_fail(e, "lane join");
  c->lane_k++;
  return CVR_OK;
}

int warm_impl(cvr_ctx* c, int max_rows, cvr_stream_t s_embed, cvr_stream_t s_dense);
int score_host_impl(cvr_ctx* c, const int32_t* h_indices, const int32_t* h_offsets, int64_t nnz, int batch,
                    const float* h_dense, float* h_scores, cvr_stream_t s_copy, cvr_stream_t s_embed,
                    cvr_stream_t s_dense);
}  // namespace

extern "C" {

int cvr_warm_graphs(cvr_ctx* c, int max_rows, cvr_stream_t s_embed, cvr_stream_t s_dense) {
  if (!c || !s_embed || !s_dense) return CVR_E_ARG;
  if (c->lanes > 1) {
    int st = ensure_lane_streams(c, (cudaStream_t)s_embed, (cudaStream_t)s_dense);
    for (int i = 0; i < c->lanes && !st; ++i) {
      st = warm_impl(c->lane(i), max_rows, c->lane_se[i], c->lane_sd[i]);
      if (st && i) st = c->fail(st, "lane %d: %s", i, c->lane_ctx[i]->err.c_str());
    }
    return st;
  }
  return warm_impl(c, max_rows, s_embed, s_dense);
}

}  // extern "C"

namespace {
int warm_impl(cvr_ctx* c, int max_rows, cvr_stream_t s_embed, cvr_stream_t s_dense) {
  int st = check_ready(c, true, true);
  if (st) return st;
  if (c->world != 1) return c->fail(CVR_E_STATE, "the executor is unsharded");
  if (max_rows < 1 || max_rows > c->max_batch) return c->fail(CVR_E_ARG, "max_rows %d outside [1, %d]", max_rows, c->max_batch);
  if (!c->use_graphs) return CVR_OK;
  bool keys = true;
  for (int t = 0; t < c->T; ++t) keys &= c->tvocab[t] > 0;
  int last = 0;
  c->bucket_rows(max_rows, &last);
  for (int slot = 0; slot < cvr_ctx::kSlots && !st; ++slot) {
    void* x0 = c->ws + c->off_x0[slot];
    c->call = c->at<CallArgs>(c->off_call[slot]);
    const bool ens = c->backbone == CVR_ENSEMBLE;
    const CUtensorMap* tm = (c->backbone == CVR_DCN_LOWRANK || c->backbone == CVR_MASKNET) ? &c->tm_x0slot[slot]
                            : ens ? &c->ens.flat_x0[slot] : nullptr;
    const CUtensorMap* tmt = ens ? &c->ens.tok_x0[slot] : nullptr;
    for (int b = 0; b <= last && !st; ++b) {
      const int rows = std::min<int64_t>((int64_t)128 << b, c->max_batch);
      // the captured kernels read their batch from the slot's call block at execution time: placeholders here
      st = run_stage(c, cvr_ctx::G_EMBED, slot, b, (cudaStream_t)s_embed, [&](cudaStream_t s) {
        return do_embed(c, nullptr, nullptr, 0, rows, nullptr, x0, s, c->embed_bps_pipe, nullptr);
      }, false);
      if (!st && keys)
        st = run_stage(c, cvr_ctx::G_EMBED_KEYS, slot, b, (cudaStream_t)s_embed, [&](cudaStream_t s) {
          return do_embed(c, nullptr, nullptr, 0, rows, nullptr, x0, s, c->embed_bps_pipe,
                          reinterpret_cast<const uint64_t*>(16));
        }, false);
      if (!st)
        st = run_stage(c, cvr_ctx::G_DENSE, slot, b, (cudaStream_t)s_dense,
                       [&](cudaStream_t s) { return do_dense(c, x0, tm, tmt, rows, nullptr, s); }, false);
    }
  }
  c->call = nullptr;
  return st;
}
}  // namespace

extern "C" {

int cvr_score(cvr_ctx* c, const int32_t* d_indices, const int32_t* d_offsets, int64_t nnz, int batch,
              const float* d_dense, float* d_scores, cvr_stream_t s_embed, cvr_stream_t s_dense) {
  if (c && c->lanes > 1)
    return lane_dispatch(c, s_embed, s_dense, [&](cvr_ctx* t, cudaStream_t se, cudaStream_t sd) {
      return score_impl(t, d_indices, nullptr, d_offsets, nnz, batch, d_dense, d_scores, se, sd);
    });
  return score_impl(c, d_indices, nullptr, d_offsets, nnz, batch, d_dense, d_scores, s_embed, s_dense);
}

int cvr_score_keys(cvr_ctx* c, const uint64_t* d_keys, const int32_t* d_offsets, int64_t nnz, int batch,
                   const float* d_dense, float* d_scores, cvr_stream_t s_embed, cvr_stream_t s_dense) {
  if (!c) return CVR_E_ARG;
  for (int t = 0; t < c->T; ++t)
    if (c->tvocab[t] <= 0) return c->fail(CVR_E_STATE, "table %d has no hash vocab (cvr_set_feature_spec)", t);
  if (nnz > 0 && !d_keys) return c->fail(CVR_E_ARG, "null keys");
  if (c->lanes > 1)
    return lane_dispatch(c, s_embed, s_dense, [&](cvr_ctx* t, cudaStream_t se, cudaStream_t sd) {
      return score_impl(t, nullptr, d_keys, d_offsets, nnz, batch, d_dense, d_scores, se, sd);
    });
  return score_impl(c, nullptr, d_keys, d_offsets, nnz, batch, d_dense, d_scores, s_embed, s_dense);
}

int cvr_score_host(cvr_ctx* c, const int32_t* h_indices, const int32_t* h_offsets, int64_t nnz, int batch,
                   const float* h_dense, float* h_scores, cvr_stream_t s_copy, cvr_stream_t s_embed,
                   cvr_stream_t s_dense) {
  if (c && c->lanes > 1)
    return lane_dispatch(c, s_embed, s_dense, [&](cvr_ctx* t, cudaStream_t se, cudaStream_t sd) {
      return score_host_impl(t, h_indices, h_offsets, nnz, batch, h_dense, h_scores, s_copy, se, sd);
    });
  return score_host_impl(c, h_indices, h_offsets, nnz, batch, h_dense, h_scores, s_copy, s_embed, s_dense);
}

}  // extern "C"

namespace {
int score_host_impl(cvr_ctx* c, const int32_t* h_indices, const int32_t* h_offsets, int64_t nnz, int batch,
                    const float* h_dense, float* h_scores, cvr_stream_t s_copy, cvr_stream_t s_embed,
                    cvr_stream_t s_dense) {
  if (!c) return CVR_E_ARG;
  int st = check_ready(c, true, true);
  if (st) return st;
  if (c->world != 1) return c->fail(CVR_E_STATE, "cvr_score_host is unsharded");
  if (batch < 0 || batch > c->max_batch) return c->fail(CVR_E_ARG, "batch %d outside [0, %d]", batch, c->max_batch);
  if (nnz < 0 || nnz > c->max_nnz) return c->fail(CVR_E_ARG, "nnz %lld outside [0, max_nnz=%lld]", (long long)nnz, (long long)c->max_nnz);
  if (!h_offsets || !h_scores || (nnz > 0 && !h_indices) || (c->F && batch && !h_dense))
    return c->fail(CVR_E_ARG, "null pointer");
  cudaStream_t sc = (cudaStream_t)s_copy, sd = (cudaStream_t)s_dense;
  const int slot = (int)(c->k % cvr_ctx::kSlots);
  cudaError_t e = cudaSuccess;
  if (c->k >= cvr_ctx::kSlots && (e = cudaStreamWaitEvent(sc, c->ev_embed[slot], 0)) != cudaSuccess)
    return c->cuda_fail(e, "wait embed(k-kSlots)");  // embed(k-kSlots) has read this staging slot
  int32_t* di = c->at<int32_t>(c->off_idx[slot]);
  int32_t* doff = c->at<int32_t>(c->off_offs[slot]);
  float* dd = c->at<float>(c->off_dense[slot]);
  float* ds = c->at<float>(c->off_scores[slot]);
  const size_t nb = (size_t)c->local_tables.size() * batch + 1;
  if (nnz && (e = cudaMemcpyAsync(di, h_indices, (size_t)nnz * 4, cudaMemcpyHostToDevice, sc)) != cudaSuccess)
    return c->cuda_fail(e, "H2D indices");
  if ((e = cudaMemcpyAsync(doff, h_offsets, nb * 4, cudaMemcpyHostToDevice, sc)) != cudaSuccess)
    return c->cuda_fail(e, "H2D offsets");
  if (c->F && batch && (e = cudaMemcpyAsync(dd, h_dense, (size_t)batch * c->F * 4, cudaMemcpyHostToDevice, sc)) != cudaSuccess)
    return c->cuda_fail(e, "H2D dense");
  if ((e = cudaEventRecord(c->ev_copy[slot], sc)) != cudaSuccess) return c->cuda_fail(e, "record copy");
  // S8: page-locked (mapped) h_scores -> the head kernel stores the scores straight into host memory over PCIe
  // (zero-copy: no D2H copy on the dense stream's critical path, measured +7.7 us per c2 step); pageable
  // memory -> device staging + a D2H copy on s_dense
  float* zc = nullptr;
  if (c->zero_copy_scores && batch) {
    cudaPointerAttributes pa{};
    if (cudaPointerGetAttributes(&pa, h_scores) == cudaSuccess && pa.type == cudaMemoryTypeHost && pa.devicePointer)
      zc = reinterpret_cast<float*>(pa.devicePointer);
    cudaGetLastError();  // (a failed query leaves a non-sticky error code)
  }
  // the embed stream sets the call block, then waits for this batch's copies (ev_copy[slot]) before the graph
  st = score_impl(c, di, nullptr, doff, nnz, batch, dd, zc ? zc : ds, s_embed, s_dense, sc);
  if (st) return st;
  if (!zc && batch && (e = cudaMemcpyAsync(h_scores, ds, (size_t)batch * 4, cudaMemcpyDeviceToHost, sd)) != cudaSuccess)
    return c->cuda_fail(e, "D2H scores");
  return CVR_OK;
}
}  // namespace

extern "C" {

int cvr_get_status(cvr_ctx* c, cvr_stream_t stream) {
  if (!c) return CVR_E_ARG;
  CVR_FORWARD_LANES(c, cvr_get_status(lc_, stream));  // every lane's sticky flag (their work is joined into stream)
  if (!c->cuda_ready) return c->fail(CVR_E_STATE, "workspace not set");
  cudaError_t e = cudaStreamSynchronize((cudaStream_t)stream);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return c->cuda_fail(e, "asynchronous CUDA error");
  int flag = 0;
  e = cudaMemcpy(&flag, c->ws + c->off_flag, 4, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && flag) e = cudaMemset(c->ws + c->off_flag, 0, 4);
  if (e != cudaSuccess) return c->cuda_fail(e, "read status flag");
  if (flag) return c->fail(CVR_E_INDEX, "device saw an out-of-range index or malformed offsets (bag zeroed)");
  return CVR_OK;
}

int cvr_shard_buffer_bytes(const cvr_ctx* c, int batch_global, size_t* send_bytes, size_t* recv_bytes) {
  if (!c || !send_bytes || !recv_bytes || batch_global < 0) return CVR_E_ARG;
  const size_t b = (size_t)batch_global * c->T_pad * c->d * elt_size(c->act);
  *send_bytes = b;
  *recv_bytes = b;
  return CVR_OK;
}

int cvr_embed_shard(cvr_ctx* c, const int32_t* d_indices, const int32_t* d_offsets, int64_t nnz, int batch_global,
                    const float* d_dense, void* d_send, void* d_x0, cvr_stream_t stream) {
  if (!c) return CVR_E_ARG;
  int st = check_ready(c, true, false);
  if (st) return st;
  if (batch_global < 0 || batch_global % c->world || batch_global / c->world > c->max_batch)
    return c->fail(CVR_E_ARG, "batch_global %d must be a multiple of world %d with B/N <= max_batch %d", batch_global,
                   c->world, c->max_batch);
  if (!d_offsets || !d_send || !d_x0 || (nnz > 0 && !d_indices) || (c->F && batch_global && !d_dense) || nnz < 0)
    return c->fail(CVR_E_ARG, "null pointer or negative nnz");
  if (c->F && !c->slot("norm/mean")->loaded) return c->fail(CVR_E_STATE, "norm/mean,std not loaded");
  EmbedArgs a = embed_args(c, d_indices, d_offsets, nnz, batch_global, d_dense, d_send, (int64_t)c->T_pad * c->d, d_x0,
                           batch_global / c->world);
  c->pbeg((cudaStream_t)stream);
  cudaError_t e = launch_embed(a, c->num_sms, (cudaStream_t)stream);
  c->pend(K_EMBED, (cudaStream_t)stream);
  if (e != cudaSuccess) return c->cuda_fail(e, "embed_shard launch");
  return CVR_OK;
}

int cvr_set_peers(cvr_ctx* c, int n, void* const* d_peer_x0, uint32_t* const* d_peer_ready,
                  uint32_t* const* d_peer_free, uint32_t* d_local_ready, uint32_t* d_local_free) {
  if (!c || !d_peer_x0 || !d_peer_ready || !d_peer_free || !d_local_ready || !d_local_free) return CVR_E_ARG;
  if (!c->cuda_ready) return c->fail(CVR_E_STATE, "cvr_set_peers before cvr_set_workspace");
  if (c->world < 2 || n != c->world) return c->fail(CVR_E_ARG, "cvr_set_peers: n must equal world_size (> 1)");
  for (int i = 0; i < 2 * n; ++i)
    if (!d_peer_x0[i]) return c->fail(CVR_E_ARG, "peer x0 slot %d: null pointer", i);
  for (int i = 0; i < n; ++i)
    if (!d_peer_ready[i] || !d_peer_free[i]) return c->fail(CVR_E_ARG, "peer %d: null flag pointer", i);
  const size_t P = sizeof(void*);
  cudaError_t e = cudaMemcpy(c->ws + c->off_peers, d_peer_x0, 2 * n * P, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(c->ws + c->off_peers + 2 * n * P, d_peer_ready, n * P, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(c->ws + c->off_peers + 3 * n * P, d_peer_free, n * P, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return c->cuda_fail(e, "cvr_set_peers");
  c->local_ready = d_local_ready;
  c->local_free = d_local_free;
  c->peers_set = true;
  return CVR_OK;
}

int cvr_embed_fused(cvr_ctx* c, const int32_t* d_indices, const int32_t* d_offsets, int64_t nnz, int batch_global,
                    const float* d_dense, void* d_x0, uint32_t epoch, cvr_stream_t stream) {
  if (!c) return CVR_E_ARG;
  int st = check_ready(c, true, false);
  if (st) return st;
  if (!c->peers_set) return c->fail(CVR_E_STATE, "cvr_embed_fused before cvr_set_peers");
  if (epoch == 0) return c->fail(CVR_E_ARG, "epoch must start at 1 and increase by one per batch");
  if (batch_global < 0 || batch_global % c->world || batch_global / c->world > c->max_batch)
    return c->fail(CVR_E_ARG, "batch_global %d must be a multiple of world %d with B/N <= max_batch %d", batch_global,
                   c->world, c->max_batch);
  if (!d_offsets || !d_x0 || (nnz > 0 && !d_indices) || (c->F && batch_global && !d_dense) || nnz < 0)
    return c->fail(CVR_E_ARG, "null pointer or negative nnz");
  if (c->F && !c->slot("norm/mean")->loaded) return c->fail(CVR_E_STATE, "norm/mean,std not loaded");
  cudaStream_t s = (cudaStream_t)stream;
  const size_t P = sizeof(void*);
  cudaError_t e;
  if (epoch > 2) {  // every owner has finished the dense stage of epoch - 2, which read the slot we now fill
    e = launch_peer_wait(c->local_free, c->world, epoch - 2, s);
    ++c->launches;
    if (e != cudaSuccess) return c->cuda_fail(e, "peer free wait launch");
  }
  EmbedArgs a = embed_args(c, d_indices, d_offsets, nnz, batch_global, d_dense, d_x0, c->x0_ld, d_x0,
                           batch_global / c->world);
  a.peer_x0 = reinterpret_cast<void* const*>(c->ws + c->off_peers + (epoch & 1) * c->world * P);
  a.world = c->world;
  a.rank = c->rank;
  a.Bl = batch_global / c->world;
  c->pbeg(s);
  e = launch_embed(a, c->num_sms, s);
  c->pend(K_EMBED, s);
  if (e != cudaSuccess) return c->cuda_fail(e, "embed_fused launch");
  e = launch_peer_signal(reinterpret_cast<uint32_t* const*>(c->ws + c->off_peers + 2 * c->world * P), c->world,
                         c->rank, epoch, s);
  ++c->launches;
  if (e != cudaSuccess) return c->cuda_fail(e, "peer ready signal launch");
  return CVR_OK;
}

int cvr_wait_peers(cvr_ctx* c, uint32_t epoch, cvr_stream_t stream) {
  if (!c) return CVR_E_ARG;
  if (!c->peers_set) return c->fail(CVR_E_STATE, "cvr_wait_peers before cvr_set_peers");
  cudaError_t e = launch_peer_wait(c->local_ready, c->world, epoch, (cudaStream_t)stream);
  ++c->launches;
  if (e != cudaSuccess) return c->cuda_fail(e, "peer wait launch");
  return CVR_OK;
}

int cvr_release_peers(cvr_ctx* c, uint32_t epoch, cvr_stream_t stream) {
  if (!c) return CVR_E_ARG;
  if (!c->peers_set) return c->fail(CVR_E_STATE, "cvr_release_peers before cvr_set_peers");
  const size_t P = sizeof(void*);
  cudaError_t e = launch_peer_signal(reinterpret_cast<uint32_t* const*>(c->ws + c->off_peers + 3 * c->world * P),
                                     c->world, c->rank, epoch, (cudaStream_t)stream);
  ++c->launches;
  if (e != cudaSuccess) return c->cuda_fail(e, "peer free signal launch");
  return CVR_OK;
}

// CUDA IPC handles name a whole allocation (cudaIpcGetMemHandle), but callers pass tensors that a caching allocator
// may have sub-allocated at an offset inside it: the handle blob carries that offset (cuMemGetAddressRange) and
// the opening side adds it back; the opened base is remembered so cvr_ipc_close_handle can unmap it.
static std::map<void*, void*> g_ipc_bases;          // opened tensor pointer -> mapped allocation base
static std::map<std::string, std::pair<void*, int>> g_ipc_maps;  // allocation handle -> (mapped base, opened tensors)
static std::mutex g_ipc_mu;                         // (the IPC entry points take no ctx: any thread may call them)

int cvr_ipc_get_handle(const void* d_ptr, void* handle) {
  if (!d_ptr || !handle) return CVR_E_ARG;
  static PFN_cuMemGetAddressRange_v3020 range = nullptr;
  if (!range) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn)
      return CVR_E_CUDA;
    range = reinterpret_cast<PFN_cuMemGetAddressRange_v3020>(fn);
  }
  CUdeviceptr base = 0;
  size_t size = 0;
  if (range(&base, &size, (CUdeviceptr)(uintptr_t)d_ptr) != CUDA_SUCCESS) return CVR_E_CUDA;
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)) != cudaSuccess) return CVR_E_CUDA;
  static_assert(sizeof(h) == 64, "CUDA IPC handles are 64 bytes");
  const int64_t off = (int64_t)((uintptr_t)d_ptr - (uintptr_t)base);
  memcpy(handle, &h, 64);
  memcpy(reinterpret_cast<uint8_t*>(handle) + 64, &off, 8);
  return CVR_OK;
}

int cvr_ipc_open_handle(const void* handle, void** d_ptr) {
  if (!handle || !d_ptr) return CVR_E_ARG;
  cudaIpcMemHandle_t h;
  int64_t off = 0;
  memcpy(&h, handle, 64);
  memcpy(&off, reinterpret_cast<const uint8_t*>(handle) + 64, 8);
  if (off < 0) return CVR_E_ARG;
  std::lock_guard<std::mutex> lk(g_ipc_mu);
  const std::string key(reinterpret_cast<const char*>(&h), 64);
  auto it = g_ipc_maps.find(key);
  void* base = nullptr;
  if (it != g_ipc_maps.end()) {  // several tensors of one allocation: one mapping, reference-counted
    base = it->second.first;
    ++it->second.second;
  } else {
    if (cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) return CVR_E_CUDA;
    g_ipc_maps[key] = {base, 1};
  }
  *d_ptr = reinterpret_cast<uint8_t*>(base) + off;
  g_ipc_bases[*d_ptr] = base;
  return CVR_OK;
}

int cvr_ipc_close_handle(void* d_ptr) {
  if (!d_ptr) return CVR_E_ARG;
  std::lock_guard<std::mutex> lk(g_ipc_mu);
  auto it = g_ipc_bases.find(d_ptr);
  if (it == g_ipc_bases.end()) return CVR_E_ARG;
  void* base = it->second;
  g_ipc_bases.erase(it);
  for (auto m = g_ipc_maps.begin(); m != g_ipc_maps.end(); ++m) {
    if (m->second.first != base) continue;
    if (--m->second.second > 0) return CVR_OK;
    g_ipc_maps.erase(m);
    return cudaIpcCloseMemHandle(base) == cudaSuccess ? CVR_OK : CVR_E_CUDA;
  }
  return CVR_E_ARG;
}

// ---- S4 through the library's own NCCL communicator ----------------------------------
int cvr_comm_unique_id(cvr_nccl_id* id) {
  if (!id) return CVR_E_ARG;
  if (!g_nccl.load()) return CVR_E_NCCL;
  return g_nccl.getUniqueId(id) == 0 ? CVR_OK : CVR_E_NCCL;
}

int cvr_comm_init(cvr_ctx* c, const cvr_nccl_id* id, int world, int rank) {
  if (!c || !id) return CVR_E_ARG;
  if (!c->cuda_ready) return c->fail(CVR_E_STATE, "cvr_comm_init before cvr_set_workspace");
  if (world != c->world || rank != c->rank)
    return c->fail(CVR_E_ARG, "cvr_comm_init(world %d, rank %d) != the ctx's world_size %d / rank %d", world, rank,
                   c->world, c->rank);
  if (c->nccl_comm) return c->fail(CVR_E_STATE, "communicator already initialised");
  if (!g_nccl.load()) return c->fail(CVR_E_NCCL, "%s", g_nccl.why.c_str());
  void* comm = nullptr;
  const int r = g_nccl.commInitRank(&comm, world, *id, rank);
  if (r != 0) return c->fail(CVR_E_NCCL, "ncclCommInitRank: %s", g_nccl.err(r));
  c->nccl_comm = comm;
  c->comm_world = world;
  c->comm_rank = rank;
  return CVR_OK;
}

int cvr_exchange(cvr_ctx* c, const void* d_send, void* d_recv, int batch_global, void* d_x0_local,
                 cvr_stream_t stream) {
  if (!c) return CVR_E_ARG;
  if (!c->cuda_ready) return c->fail(CVR_E_STATE, "workspace not set");
  if (!c->nccl_comm) return c->fail(CVR_E_STATE, "cvr_exchange before cvr_comm_init");
  if (!d_send || !d_recv || !d_x0_local || batch_global < 0 || batch_global % c->world ||
      batch_global / c->world > c->max_batch)
    return c->fail(CVR_E_ARG, "bad arguments (batch_global %d, world %d)", batch_global, c->world);
  cudaStream_t s = (cudaStream_t)stream;
  const size_t chunk = (size_t)(batch_global / c->world) * c->T_pad * c->d * elt_size(c->act);
  if (chunk) {
    // chunk dst of d_send (destination-major [dst][b_local][t_slot][d]) -> rank dst; chunk src of d_recv <- rank src
    int r = g_nccl.groupStart();
    for (int p = 0; p < c->world && r == 0; ++p) {
      r = g_nccl.send(reinterpret_cast<const uint8_t*>(d_send) + p * chunk, chunk, kNcclUint8, p, c->nccl_comm, s);
      if (r == 0) r = g_nccl.recv(reinterpret_cast<uint8_t*>(d_recv) + p * chunk, chunk, kNcclUint8, p, c->nccl_comm, s);
    }
    const int r2 = g_nccl.groupEnd();
    if (r != 0 || r2 != 0) return c->fail(CVR_E_NCCL, "grouped ncclSend/ncclRecv: %s", g_nccl.err(r ? r : r2));
  }
  ++c->launches;  // (the NCCL kernel)
  c->pbeg(s);
  cudaError_t e = launch_unpack(d_recv, d_x0_local, c->x0_ld, c->world, batch_global / c->world, c->T_pad, c->T, c->d,
                                c->act, s);
  c->pend(K_UNPACK, s);
  if (e != cudaSuccess) return c->cuda_fail(e, "unpack launch");
  return CVR_OK;
}

int cvr_repeat_kernel(cvr_ctx* c, const char* role, int reps, const void* d_x0, int batch, cvr_stream_t stream,
                      int* n_launched) {
  if (!c || !role || reps < 1 || !n_launched) return CVR_E_ARG;
  int st = check_ready(c, false, true);
  if (st) return st;
  if (c->backbone == CVR_DCN_FULL) return c->fail(CVR_E_UNSUPPORTED, "cvr_repeat_kernel: tcgen05 GEMM roles only");
  int kid = -1;
  for (int k = 0; k < K_COUNT; ++k)
    if (!strcmp(role, kKernelNames[k])) kid = k;
  if (kid < 0 || strncmp(role, "gemm_", 5) != 0) return c->fail(CVR_E_ARG, "unknown GEMM role '%s'", role);
  float* scores = c->at<float>(c->off_scores[0]);  // (the head writes into the ctx's own score staging)
  const int64_t l0 = c->launches;
  c->only_kid = kid;
  c->only_reps = reps;
  st = cvr_dense(c, d_x0, batch, scores, stream);
  c->only_kid = -1;
  c->only_reps = 1;
  *n_launched = (int)(c->launches - l0);
  return st;
}

int cvr_call_info(const cvr_ctx* c, int slot, cvr_call_record* out) {
  if (!c || !out || slot < 0 || slot >= cvr_ctx::kSlots * c->lanes) return CVR_E_ARG;
  if (!c->cuda_ready) return CVR_E_STATE;
  if (slot >= cvr_ctx::kSlots) {  // lane slot / kSlots, its slot % kSlots
    const int st = cvr_call_info(c->lane_ctx[slot / cvr_ctx::kSlots], slot % cvr_ctx::kSlots, out);
    if (st == CVR_OK)
      for (int i = 0; i < c->lanes; ++i) out->graph_captures += i != slot / cvr_ctx::kSlots ? c->lane(i)->graph_captures : 0;
    return st;
  }
  CallArgs v{};
  if (cudaMemcpy(&v, c->ws + c->off_call[slot], sizeof v, cudaMemcpyDeviceToHost) != cudaSuccess) return CVR_E_CUDA;
  out->d_indices = v.indices;
  out->d_keys = v.keys;
  out->d_offsets = v.offsets;
  out->d_dense = v.dense;
  out->d_scores = v.scores;
  out->nnz = v.nnz;
  out->batch = v.B;
  out->graph_captures = 0;
  for (int i = 0; i < c->lanes; ++i) out->graph_captures += i ? c->lane_ctx[i]->graph_captures : c->graph_captures;
  return CVR_OK;
}

int cvr_unpack_shard(cvr_ctx* c, const void* d_recv, int batch_global, void* d_x0, cvr_stream_t stream) {
  if (!c) return CVR_E_ARG;
  if (!c->cuda_ready) return c->fail(CVR_E_STATE, "workspace not set");
  if (!d_recv || !d_x0 || batch_global < 0 || batch_global % c->world) return c->fail(CVR_E_ARG, "bad arguments");
  c->pbeg((cudaStream_t)stream);
  cudaError_t e = launch_unpack(d_recv, d_x0, c->x0_ld, c->world, batch_global / c->world, c->T_pad, c->T, c->d, c->act,
                                (cudaStream_t)stream);
  c->pend(K_UNPACK, (cudaStream_t)stream);
  if (e != cudaSuccess) return c->cuda_fail(e, "unpack launch");
  return CVR_OK;
}

int cvr_launch_count(const cvr_ctx* c, int64_t* n) {
  if (!c || !n) return CVR_E_ARG;
  *n = c->launches;
  for (int i = 1; i < c->lanes; ++i) *n += c->lane_ctx[i]->launches;
  return CVR_OK;
}

int cvr_profile_begin(cvr_ctx* c, int max_launches) {
  if (!c || max_launches < 0) return CVR_E_ARG;
  if (!c->cuda_ready) return c->fail(CVR_E_STATE, "workspace not set");
  while (c->prof_ev.size() < (size_t)max_launches * 2) {
    cudaEvent_t ev;
    cudaError_t e = cudaEventCreate(&ev);
    if (e != cudaSuccess) return c->cuda_fail(e, "profile event create");
    c->prof_ev.push_back(ev);
  }
  c->prof_kid.assign((size_t)max_launches, 0);
  c->prof_cap = (size_t)max_launches;
  c->prof_n = 0;
  c->prof_on = true;
  return CVR_OK;
}

int cvr_profile_end(cvr_ctx* c, cvr_kernel_stat* out, int max_out, int* n_out) {
  if (!c || !n_out || (max_out > 0 && !out)) return CVR_E_ARG;
  c->prof_on = false;

  cvr_kernel_stat agg[K_COUNT];
  memset(agg, 0, sizeof agg);
  for (size_t i = 0; i < c->prof_n; ++i) {
    cudaError_t e = cudaEventSynchronize(c->prof_ev[2 * i + 1]);
    float ms = 0.f;
    if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, c->prof_ev[2 * i], c->prof_ev[2 * i + 1]);
    if (e != cudaSuccess) return c->cuda_fail(e, "profile read");
    cvr_kernel_stat& a = agg[c->prof_kid[i]];
    if (a.launches == 0 || ms < a.min_ms) a.min_ms = ms;
    if (a.launches == 0 || ms > a.max_ms) a.max_ms = ms;
    a.total_ms += ms;
    a.launches++;
  }
  int n = 0;
  for (int k = 0; k < K_COUNT; ++k) {
    if (!agg[k].launches) continue;
    if (n < max_out) {
      out[n] = agg[k];
      snprintf(out[n].name, sizeof out[n].name, "%s", kKernelNames[k]);
    }
    ++n;
  }
  *n_out = n;
  c->prof_n = 0;
  return CVR_OK;
}

int cvr_gemm_bf16(const void* d_A, int64_t lda, const void* d_B, int64_t ldb, void* d_C, int64_t ldc, int M, int N,
                  int K, int epi, const float* d_bias, int bn, cvr_stream_t stream) {
  const bool pair = (epi & 0x100) != 0;
  epi &= 0xFF;
  if (!d_A || !d_B || !d_C || M < 0 || N <= 0 || K <= 0 || (epi == 1 && !d_bias)) return CVR_E_ARG;
  if (d_bias && (reinterpret_cast<uintptr_t>(d_bias) & 15)) return CVR_E_ARG;  // read as float4
  if (epi != 0 && epi != 1) return CVR_E_ARG;
  if (K % 64 || N % bn || (bn != 64 && bn != 128 && bn != 256 && !(bn == 192 && epi == 0 && !pair)) || lda < K || ldb < K || ldc < N || (lda | ldb | ldc) & 7)
    return CVR_E_UNSUPPORTED;
  if (M == 0) return CVR_OK;
  const char* er = nullptr;
  CUtensorMap ta, tb, tc;
  if (encode_tmap_bf16(&ta, d_A, M, K, lda, 128, &er) || encode_tmap_bf16(&tb, d_B, N, K, ldb, pair ? bn / 2 : bn, &er) ||
      encode_tmap_bf16(&tc, d_C, M, N, ldc, 32, &er))
    return CVR_E_CUDA;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  GemmArgs a{};
  a.tmA = &ta;
  a.tmB = &tb;
  a.tmOut = &tc;
  a.bias = d_bias;
  a.M = M;
  a.N = N;
  a.K = K;
  a.BN = bn;
  a.epi = epi == 0 ? EPI_STORE : EPI_BIAS_RELU;
  a.num_sms = sms;
  a.pdl = false;
  a.cta_pair = pair;
  return launch_gemm_bf16(a, (cudaStream_t)stream) == cudaSuccess ? CVR_OK : CVR_E_CUDA;
}

int cvr_set_option(cvr_ctx* c, const char* key, int64_t value) {
  if (!c || !key) return CVR_E_ARG;
  if (!strcmp(key, "lanes")) {
    if (value < 1 || value > cvr_ctx::kMaxLanes) return c->fail(CVR_E_ARG, "lanes must be in [1, %d]", cvr_ctx::kMaxLanes);
    if (c->ws) return c->fail(CVR_E_STATE, "lanes must be set before cvr_set_workspace");
    if (c->world != 1 && value > 1) return c->fail(CVR_E_STATE, "executor lanes are unsharded (world_size 1)");
    for (int i = (int)value; i < cvr_ctx::kMaxLanes; ++i)
      if (c->lane_ctx[i]) {
        cvr_destroy(c->lane_ctx[i]);
        c->lane_ctx[i] = nullptr;
      }
    for (int i = 1; i < (int)value; ++i) {
      if (c->lane_ctx[i]) continue;
      cvr_ctx* t = nullptr;
      const int st = cvr_create(&c->desc, &t);
      if (st != CVR_OK) {
        if (t) cvr_destroy(t);
        return c->fail(st, "lane %d: create failed", i);
      }
      copy_options(t, c);
      c->lane_ctx[i] = t;
    }
    c->lanes = (int)value;
    return CVR_OK;
  }
  CVR_FORWARD_LANES(c, cvr_set_option(lc_, key, value));
  // every option below changes what the executor's graphs would launch: drop them (recaptured at next use)
  auto replan = [&]() -> int {
    c->drop_graphs();
    if (!c->weights_loaded) return CVR_OK;
    if (c->backbone == CVR_DCN_LOWRANK) return encode_plan(c);
    if (c->backbone == CVR_ENSEMBLE) return encode_plan_ensemble(c);
    return CVR_OK;
  };
  auto flag = [&](bool& f) { f = value != 0; return replan(); };
  if (!strcmp(key, "graphs")) return flag(c->use_graphs);
  if (!strcmp(key, "pdl")) return flag(c->pdl);
  if (!strcmp(key, "prefetch_b")) return flag(c->prefetch_b);
  if (!strcmp(key, "pair")) return flag(c->pair_ens);
  if (!strcmp(key, "f32_tma_store")) return flag(c->f32_tma_store);
  if (!strcmp(key, "ens_xv_wave")) return flag(c->ens_xv_wave);
  if (!strcmp(key, "ens_ffn_fused")) return flag(c->ens_ffn_fused);
  if (!strcmp(key, "ens_fused_attn")) return flag(c->ens_fused_attn);
  if (!strcmp(key, "ens_attn_tc")) return flag(c->ens_attn_tc);
  if (!strcmp(key, "mask_grouped")) return flag(c->mask_grouped);
  if (!strcmp(key, "zero_copy_scores")) {
    c->zero_copy_scores = value != 0;
    return CVR_OK;
  }
  if (!strcmp(key, "embed_bps")) {
    if (value < 0 || value > 64) return c->fail(CVR_E_ARG, "embed_bps must be in [0, 64]");
    c->embed_bps_pipe = (int)value;
    return replan();
  }
  if (!strcmp(key, "ens_u_bn")) {
    if (value != 64 && value != 128) return c->fail(CVR_E_ARG, "ens_u_bn must be 64 or 128");
    c->ens_u_bn = (int)value;
    return replan();
  }
  if (!strcmp(key, "xv_bn")) {
    if (value != 0 && value != 64 && value != 128 && value != 256) return c->fail(CVR_E_ARG, "xv_bn: 0, 64, 128 or 256");
    c->xv_bn = (int)value;
    return replan();
  }
  if (!strcmp(key, "u_bn")) {
    if (value != 64 && value != 192) return c->fail(CVR_E_ARG, "u_bn must be 64 or 192");
    c->u_bn = (int)value;
    return replan();
  }
  if (!strcmp(key, "epw")) {
    if (value < 0 || value > 2) return c->fail(CVR_E_ARG, "epw must be 0, 1 or 2");
    c->epw_mode = (int)value;
    return replan();
  }
  return c->fail(CVR_E_ARG, "unknown option '%s'", key);
}

int cvr_concat_requests(int n_req, int n_tables, int n_dense, const int* n_items, const int32_t* const* h_offsets,
                        const int32_t* const* h_indices, const float* const* h_dense, int out_batch_cap,
                        int32_t* out_offsets, int32_t* out_indices, int64_t out_indices_cap, float* out_dense,
                        int64_t* out_nnz) {
  if (n_req < 0 || n_tables <= 0 || n_dense < 0 || !n_items || !h_offsets || !h_indices || !out_offsets ||
      !out_indices || !out_nnz || (n_dense && (!h_dense || !out_dense)))
    return CVR_E_ARG;
  int64_t B = 0;
  for (int r = 0; r < n_req; ++r) {
    if (n_items[r] < 0 || !h_offsets[r]) return CVR_E_ARG;
    B += n_items[r];
  }
  if (B > out_batch_cap) return CVR_E_NOMEM;
  // table-major: for t, for request r, for item i: bag (t, r, i)
  int64_t pos = 0, bag = 0;
  out_offsets[0] = 0;
  for (int t = 0; t < n_tables; ++t) {
    for (int r = 0; r < n_req; ++r) {
      const int n = n_items[r];
      const int32_t* off = h_offsets[r] + (int64_t)t * n;
      const int32_t lo = off[0], hi = off[n];
      if (lo < 0 || hi < lo) return CVR_E_INDEX;
      for (int i = 0; i < n; ++i)  // every bag inside [lo, hi], non-decreasing (else the copy below reads out of range)
        if (off[i + 1] < off[i]) return CVR_E_INDEX;
      const int64_t len = hi - lo;
      if (pos + len > out_indices_cap) return CVR_E_NOMEM;
      if (len) memcpy(out_indices + pos, h_indices[r] + lo, (size_t)len * 4);
      for (int i = 0; i < n; ++i) out_offsets[++bag] = (int32_t)(pos + (off[i + 1] - lo));
      pos += len;
    }
  }
  if (n_dense) {
    int64_t row = 0;
    for (int r = 0; r < n_req; ++r) {
      memcpy(out_dense + row * n_dense, h_dense[r], (size_t)n_items[r] * n_dense * 4);
      row += n_items[r];
    }
  }
  *out_nnz = pos;
  return CVR_OK;
}

int cvr_gather_items(int n_tables, int n_dense, int64_t pool_size, const int32_t* pool_offsets,
                     const int32_t* pool_indices, const float* pool_dense, int n, const int32_t* item_ids,
                     int out_batch_cap, int32_t* out_offsets, int32_t* out_indices, int64_t out_indices_cap,
                     float* out_dense, int64_t* out_nnz) {
  if (n_tables <= 0 || n_dense < 0 || pool_size <= 0 || n < 0 || !pool_offsets || !pool_indices || !item_ids ||
      !out_offsets || !out_indices || !out_nnz || (n_dense && (!pool_dense || !out_dense)))
    return CVR_E_ARG;
  if (n > out_batch_cap) return CVR_E_NOMEM;  // out_offsets [T * cap + 1] and out_dense [cap, F] would overflow
  for (int i = 0; i < n; ++i)
    if (item_ids[i] < 0 || item_ids[i] >= pool_size) return CVR_E_INDEX;
  // pass 1: bag lengths -> per-table totals; pass 2: copy at the prefix offsets.  The pool reads are random
  // (item ids) and latency-bound, so both passes prefetch the offsets PF items ahead (and pass 2 the index runs of
  // items PF/2 ahead, whose offsets are cached by then).  Batches below 2048 items stay on the calling thread: an
  // OpenMP region's barrier waits for its slowest member, and on the 16-core GPU host a team member descheduled
  // for a few ms showed up as 2-11 ms outliers of single gathers (cvr_serve_stats.max_gather_s) at low load
  constexpr int PF = 16;
  const bool par = n >= 2048;
  // (large batches: the team leaves 4 cores to the polling thread's neighbours -- CUDA driver threads, the OS)
  const int nth = std::max(1, omp_get_max_threads() - 4);
  std::vector<int64_t> tot(n_tables + 1, 0);
  int bad = 0;
#pragma omp parallel for schedule(static) reduction(| : bad) if (par) num_threads(nth)
  for (int t = 0; t < n_tables; ++t) {
    const int32_t* off = pool_offsets + (int64_t)t * pool_size;
    int64_t s = 0;
    for (int i = 0; i < n; ++i) {
      if (i + PF < n) __builtin_prefetch(off + item_ids[i + PF]);
      const int64_t it = item_ids[i];
      const int32_t len = off[it + 1] - off[it];
      bad |= len < 0;
      s += len;
    }
    tot[t + 1] = s;
  }
  if (bad) return CVR_E_INDEX;
  for (int t = 0; t < n_tables; ++t) tot[t + 1] += tot[t];
  if (tot[n_tables] > out_indices_cap) return CVR_E_NOMEM;
  out_offsets[0] = 0;
#pragma omp parallel for schedule(static) if (par) num_threads(nth)
  for (int t = 0; t < n_tables; ++t) {
    const int32_t* off = pool_offsets + (int64_t)t * pool_size;
    int64_t pos = tot[t];
    for (int i = 0; i < n; ++i) {
      if (i + PF < n) __builtin_prefetch(off + item_ids[i + PF]);
      if (i + PF / 2 < n) __builtin_prefetch(pool_indices + off[item_ids[i + PF / 2]]);
      const int64_t it = item_ids[i];
      const int32_t lo = off[it], hi = off[it + 1];
      for (int32_t q = lo; q < hi; ++q) out_indices[pos++] = pool_indices[q];
      out_offsets[(int64_t)t * n + i + 1] = (int32_t)pos;
    }
  }
#pragma omp parallel for schedule(static) if (par) num_threads(nth)
  for (int i = 0; i < (n_dense ? n : 0); ++i) {
    if (i + PF < n) __builtin_prefetch(pool_dense + (int64_t)item_ids[i + PF] * n_dense);
    memcpy(out_dense + (int64_t)i * n_dense, pool_dense + (int64_t)item_ids[i] * n_dense, (size_t)n_dense * 4);
  }
  *out_nnz = tot[n_tables];
  return CVR_OK;
}

int cvr_text_ngram_keys(int n_texts, const char* const* texts, const int32_t* lens, int n, uint64_t* out_keys,
                        int64_t out_cap, int32_t* out_offsets, int64_t* out_nnz) {
  if (n_texts < 0 || n < 1 || n > 8 || !out_offsets || !out_nnz || (n_texts > 0 && (!texts || !lens)))
    return CVR_E_ARG;
  int64_t pos = 0;
  out_offsets[0] = 0;
  for (int i = 0; i < n_texts; ++i) {
    const int32_t L = lens[i];
    if (L < 0 || (L > 0 && !texts[i])) return CVR_E_ARG;
    const unsigned char* t = reinterpret_cast<const unsigned char*>(texts[i]);
    for (int32_t k = 0; k + n <= L; ++k) {  // overlapping n-byte grams, packed big-endian (A29)
      if (pos >= out_cap) return CVR_E_NOMEM;
      uint64_t key = 0;
      for (int b = 0; b < n; ++b) key = (key << 8) | t[k + b];
      out_keys[pos++] = key;
    }
    if (pos > INT32_MAX) return CVR_E_NOMEM;
    out_offsets[i + 1] = (int32_t)pos;
  }
  *out_nnz = pos;
  return CVR_OK;
}

int cvr_truncate_bags(int n_bags, const int32_t* offsets, const uint64_t* keys, int max_len, int32_t* out_offsets,
                      uint64_t* out_keys, int64_t* out_nnz) {
  if (n_bags < 0 || max_len < 0 || !offsets || !out_offsets || !out_nnz) return CVR_E_ARG;
  int64_t pos = 0;
  out_offsets[0] = 0;
  for (int i = 0; i < n_bags; ++i) {
    const int32_t lo = offsets[i], hi = offsets[i + 1];
    if (hi < lo) return CVR_E_INDEX;
    const int32_t keep_lo = hi - lo > max_len ? hi - max_len : lo;  // the most recent max_len keys
    for (int32_t q = keep_lo; q < hi; ++q) out_keys[pos++] = keys[q];
    out_offsets[i + 1] = (int32_t)pos;
  }
  *out_nnz = pos;
  return CVR_OK;
}

}  // extern "C"
