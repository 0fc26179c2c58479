"""ctypes binding of libcvr.so (include/cvr.h).  Argument marshalling only: every step of the
path runs in the library's kernels; torch tensors are passed as raw pointers and streams as
cudaStream_t handles."""
from __future__ import annotations

import ctypes
import os
from typing import Dict, Optional, Sequence

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
lib_path = os.environ.get("CVR_LIB") or os.path.join(HERE, "libcvr.so")  # CVR_LIB: A/B of two builds (experiments)

CVR_F32, CVR_BF16, CVR_F16 = 0, 1, 2
CVR_DCN_FULL, CVR_DCN_LOWRANK, CVR_ENSEMBLE, CVR_MASKNET = 0, 1, 2, 3
CVR_E_INDEX = 5
_DT = {"f32": CVR_F32, "bf16": CVR_BF16, "f16": CVR_F16}
_TORCH_DT = {torch.float32: CVR_F32, torch.bfloat16: CVR_BF16, torch.float16: CVR_F16}
_BACKBONE = {"dcn_full": CVR_DCN_FULL, "dcn_lowrank": CVR_DCN_LOWRANK, "ensemble": CVR_ENSEMBLE,
             "masknet": CVR_MASKNET}

_c_i64p = ctypes.POINTER(ctypes.c_int64)
_c_ip = ctypes.POINTER(ctypes.c_int)
_vp = ctypes.c_void_p


class cvr_model_desc(ctypes.Structure):
    _fields_ = [
        ("n_tables", ctypes.c_int), ("rows", _c_i64p), ("dim", ctypes.c_int), ("emb_dtype", ctypes.c_int),
        ("n_dense", ctypes.c_int), ("act_dtype", ctypes.c_int), ("backbone", ctypes.c_int),
        ("n_cross", ctypes.c_int), ("cross_rank", ctypes.c_int), ("n_mlp", ctypes.c_int), ("mlp_dims", _c_ip),
        ("n_heads", ctypes.c_int), ("ffn_dim", ctypes.c_int), ("max_batch", ctypes.c_int),
        ("max_nnz", ctypes.c_int64), ("world_size", ctypes.c_int), ("rank", ctypes.c_int),
        ("cross_width", ctypes.c_int), ("n_parallel", ctypes.c_int),
    ]


class cvr_nccl_id(ctypes.Structure):
    _fields_ = [("internal", ctypes.c_char * 128)]


class cvr_call_record(ctypes.Structure):
    _fields_ = [("d_indices", _vp), ("d_keys", _vp), ("d_offsets", _vp), ("d_dense", _vp), ("d_scores", _vp),
                ("nnz", ctypes.c_int64), ("batch", ctypes.c_int), ("graph_captures", ctypes.c_int64)]


class cvr_serve_config(ctypes.Structure):
    _fields_ = [("window_s", ctypes.c_double), ("max_items", ctypes.c_int), ("max_requests", ctypes.c_int),
                ("queue_capacity", ctypes.c_int), ("host_slots", ctypes.c_int), ("max_nnz", ctypes.c_int64),
                ("abort_after_s", ctypes.c_double)]


class cvr_serve_stats(ctypes.Structure):
    _fields_ = [("rejected", ctypes.c_int64), ("aborted", ctypes.c_int), ("items_served", ctypes.c_int64),
                ("host_dispatch_s", ctypes.c_double), ("wall_s", ctypes.c_double), ("max_dispatch_s", ctypes.c_double),
                ("max_gather_s", ctypes.c_double),
                ("loop_gaps_1ms", ctypes.c_int64)]


IPC_HANDLE_BYTES = 72
EXECUTOR_SLOTS = 2  # CVR_EXECUTOR_SLOTS: batch k of cvr_score / cvr_score_host uses x0 slot k % 2  # CVR_IPC_HANDLE_BYTES: CUDA IPC handle of the allocation + the tensor's offset inside it


class cvr_kernel_stat(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char * 32), ("launches", ctypes.c_int64), ("total_ms", ctypes.c_double),
                ("min_ms", ctypes.c_double), ("max_ms", ctypes.c_double)]


# (name, restype, argtypes) -- mirrors include/cvr.h
_SIGS = [
    ("cvr_create", ctypes.c_int, [ctypes.POINTER(cvr_model_desc), ctypes.POINTER(_vp)]),
    ("cvr_destroy", ctypes.c_int, [_vp]),
    ("cvr_last_error", ctypes.c_char_p, [_vp]),
    ("cvr_status_string", ctypes.c_char_p, [ctypes.c_int]),
    ("cvr_version", ctypes.c_char_p, []),
    ("cvr_workspace_bytes", ctypes.c_int, [_vp, ctypes.POINTER(ctypes.c_size_t)]),
    ("cvr_set_workspace", ctypes.c_int, [_vp, _vp, ctypes.c_size_t]),
    ("cvr_x0_layout", ctypes.c_int, [_vp, _c_ip, _c_ip]),
    ("cvr_load_tables", ctypes.c_int, [_vp, ctypes.c_int, _c_ip, ctypes.POINTER(_vp), _c_i64p]),
    ("cvr_load_weights", ctypes.c_int,
     [_vp, ctypes.c_int, ctypes.POINTER(ctypes.c_char_p), ctypes.POINTER(_vp), _c_ip, _c_ip, _c_i64p]),
    ("cvr_embed", ctypes.c_int, [_vp, _vp, _vp, ctypes.c_int64, ctypes.c_int, _vp, _vp, _vp]),
    ("cvr_dense", ctypes.c_int, [_vp, _vp, ctypes.c_int, _vp, _vp]),
    ("cvr_score", ctypes.c_int, [_vp, _vp, _vp, ctypes.c_int64, ctypes.c_int, _vp, _vp, _vp, _vp]),
    ("cvr_warm_graphs", ctypes.c_int, [_vp, ctypes.c_int, _vp, _vp]),
    ("cvr_score_host", ctypes.c_int, [_vp, _vp, _vp, ctypes.c_int64, ctypes.c_int, _vp, _vp, _vp, _vp, _vp]),
    ("cvr_get_status", ctypes.c_int, [_vp, _vp]),
    ("cvr_shard_buffer_bytes", ctypes.c_int, [_vp, ctypes.c_int, ctypes.POINTER(ctypes.c_size_t),
                                              ctypes.POINTER(ctypes.c_size_t)]),
    ("cvr_embed_shard", ctypes.c_int, [_vp, _vp, _vp, ctypes.c_int64, ctypes.c_int, _vp, _vp, _vp, _vp]),
    ("cvr_unpack_shard", ctypes.c_int, [_vp, _vp, ctypes.c_int, _vp, _vp]),
    ("cvr_set_peers", ctypes.c_int, [_vp, ctypes.c_int, ctypes.POINTER(_vp), ctypes.POINTER(_vp), ctypes.POINTER(_vp),
                                     _vp, _vp]),
    ("cvr_embed_fused", ctypes.c_int, [_vp, _vp, _vp, ctypes.c_int64, ctypes.c_int, _vp, _vp, ctypes.c_uint32, _vp]),
    ("cvr_wait_peers", ctypes.c_int, [_vp, ctypes.c_uint32, _vp]),
    ("cvr_release_peers", ctypes.c_int, [_vp, ctypes.c_uint32, _vp]),
    ("cvr_ipc_get_handle", ctypes.c_int, [_vp, _vp]),
    ("cvr_ipc_open_handle", ctypes.c_int, [_vp, ctypes.POINTER(_vp)]),
    ("cvr_ipc_close_handle", ctypes.c_int, [_vp]),
    ("cvr_comm_unique_id", ctypes.c_int, [ctypes.POINTER(cvr_nccl_id)]),
    ("cvr_comm_init", ctypes.c_int, [_vp, ctypes.POINTER(cvr_nccl_id), ctypes.c_int, ctypes.c_int]),
    ("cvr_exchange", ctypes.c_int, [_vp, _vp, _vp, ctypes.c_int, _vp, _vp]),
    ("cvr_call_info", ctypes.c_int, [_vp, ctypes.c_int, ctypes.POINTER(cvr_call_record)]),
    ("cvr_repeat_kernel", ctypes.c_int, [_vp, ctypes.c_char_p, ctypes.c_int, _vp, ctypes.c_int, _vp, _c_ip]),
    ("cvr_gemm_bf16", ctypes.c_int, [_vp, ctypes.c_int64, _vp, ctypes.c_int64, _vp, ctypes.c_int64, ctypes.c_int,
                                     ctypes.c_int, ctypes.c_int, ctypes.c_int, _vp, ctypes.c_int, _vp]),
    ("cvr_set_option", ctypes.c_int, [_vp, ctypes.c_char_p, ctypes.c_int64]),
    ("cvr_concat_requests", ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, _c_ip, ctypes.POINTER(_vp),
                                           ctypes.POINTER(_vp), ctypes.POINTER(_vp), ctypes.c_int, _vp, _vp,
                                           ctypes.c_int64, _vp, _c_i64p]),
    ("cvr_gather_items", ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int64, _vp, _vp, _vp, ctypes.c_int, _vp,
                                        ctypes.c_int, _vp, _vp, ctypes.c_int64, _vp, _c_i64p]),
    ("cvr_serve_trace", ctypes.c_int, [_vp, ctypes.POINTER(cvr_serve_config), ctypes.c_int, ctypes.c_int,
                                       ctypes.c_int64, _vp, _vp, _vp, ctypes.c_int, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                                       _c_ip, ctypes.POINTER(cvr_serve_stats), _vp, _vp, _vp]),
    ("cvr_batcher_simulate", ctypes.c_int, [ctypes.c_int, _vp, _vp, ctypes.c_double, ctypes.c_int, ctypes.c_int,
                                            ctypes.c_int, ctypes.c_double, ctypes.c_double, _vp, _vp, _vp, _c_ip]),
    ("cvr_set_feature_spec", ctypes.c_int, [_vp, ctypes.c_int, _c_i64p, _c_ip]),
    ("cvr_embed_keys", ctypes.c_int, [_vp, _vp, _vp, ctypes.c_int64, ctypes.c_int, _vp, _vp, _vp]),
    ("cvr_score_keys", ctypes.c_int, [_vp, _vp, _vp, ctypes.c_int64, ctypes.c_int, _vp, _vp, _vp, _vp]),
    ("cvr_text_ngram_keys", ctypes.c_int, [ctypes.c_int, ctypes.POINTER(ctypes.c_char_p), _c_ip, ctypes.c_int, _vp,
                                           ctypes.c_int64, _vp, _c_i64p]),
    ("cvr_truncate_bags", ctypes.c_int, [ctypes.c_int, _vp, _vp, ctypes.c_int, _vp, _vp, _c_i64p]),
    ("cvr_launch_count", ctypes.c_int, [_vp, _c_i64p]),
    ("cvr_profile_begin", ctypes.c_int, [_vp, ctypes.c_int]),
    ("cvr_profile_end", ctypes.c_int, [_vp, ctypes.POINTER(cvr_kernel_stat), ctypes.c_int, _c_ip]),
]

_lib = None


def lib() -> ctypes.CDLL:
    """Load libcvr.so (fails loudly if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(lib_path):
            raise ImportError(f"{lib_path} not built: run `python -m paper_2605_29232_b200.build` "
                              "(there is no CPU fallback)")
        L = ctypes.CDLL(lib_path)
        for name, res, args in _SIGS:
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def status_string(st: int) -> str:
    return lib().cvr_status_string(st).decode()


class CvrError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{status_string(status)}: {msg}")
        self.status = status


def _ptr(t: Optional[torch.Tensor]) -> Optional[int]:
    return None if t is None else t.data_ptr()


def _stream(s) -> Optional[int]:
    if s is None:
        return torch.cuda.current_stream().cuda_stream
    if isinstance(s, torch.cuda.Stream):
        return s.cuda_stream
    return int(s)


def gemm_bf16(A: torch.Tensor, B: torch.Tensor, C: Optional[torch.Tensor] = None, bias: Optional[torch.Tensor] = None,
              bn: int = 64, stream=None, pair: bool = False) -> torch.Tensor:
    """C = A @ B^T (bf16, fp32 accumulate) [+ bias, ReLU] on libcvr's tcgen05 GEMM (cvr_gemm_bf16)."""
    M, K = A.shape
    N = B.shape[0]
    C = torch.empty(M, N, dtype=torch.bfloat16, device=A.device) if C is None else C
    st = lib().cvr_gemm_bf16(A.data_ptr(), A.stride(0), B.data_ptr(), B.stride(0), C.data_ptr(), C.stride(0), M, N, K,
                             (0 if bias is None else 1) | (0x100 if pair else 0), _ptr(bias), bn, _stream(stream))
    if st != 0:
        raise CvrError(st, "cvr_gemm_bf16")
    return C


def ipc_get_handle(ptr: int) -> bytes:
    """cvr_ipc_get_handle: the CUDA IPC handle of the allocation holding ``ptr`` + ptr's offset in it (72 bytes)."""
    buf = ctypes.create_string_buffer(IPC_HANDLE_BYTES)
    st = lib().cvr_ipc_get_handle(ptr, buf)
    if st != 0:
        raise CvrError(st, "cvr_ipc_get_handle")
    return buf.raw


def ipc_open_handle(handle: bytes) -> int:
    """cvr_ipc_open_handle: map another process's allocation; returns the device pointer of the tensor."""
    p = _vp()
    st = lib().cvr_ipc_open_handle(ctypes.create_string_buffer(handle, IPC_HANDLE_BYTES), ctypes.byref(p))
    if st != 0:
        raise CvrError(st, "cvr_ipc_open_handle")
    return p.value


def ipc_close_handle(ptr: int) -> None:
    st = lib().cvr_ipc_close_handle(ptr)
    if st != 0:
        raise CvrError(st, "cvr_ipc_close_handle")


def comm_unique_id() -> bytes:
    """cvr_comm_unique_id: a fresh NCCL unique id (128 bytes), to be broadcast to every rank."""
    uid = cvr_nccl_id()
    st = lib().cvr_comm_unique_id(ctypes.byref(uid))
    if st != 0:
        raise CvrError(st, "cvr_comm_unique_id (NCCL unavailable?)")
    return ctypes.string_at(ctypes.addressof(uid), 128)  # (uid.internal would stop at the first NUL byte)


def text_ngram_keys(texts, n: int):
    """cvr_text_ngram_keys (host): byte strings -> (keys uint64 ndarray, offsets int32 ndarray)."""
    import numpy as np
    cap = sum(max(0, len(t) - n + 1) for t in texts)
    arr = (ctypes.c_char_p * max(1, len(texts)))(*texts)
    lens = (ctypes.c_int * max(1, len(texts)))(*[len(t) for t in texts])
    keys = np.zeros(max(1, cap), np.uint64)
    off = np.zeros(len(texts) + 1, np.int32)
    nnz = ctypes.c_int64()
    st = lib().cvr_text_ngram_keys(len(texts), arr, lens, n, keys.ctypes.data, cap, off.ctypes.data, ctypes.byref(nnz))
    if st != 0:
        raise CvrError(st, "cvr_text_ngram_keys")
    return keys[:nnz.value], off


def truncate_bags(keys, offsets, max_len: int):
    """cvr_truncate_bags (host): keep the most recent max_len keys of each bag."""
    import numpy as np
    keys = np.ascontiguousarray(keys, np.uint64)
    offsets = np.ascontiguousarray(offsets, np.int32)
    n = len(offsets) - 1
    out_k = np.zeros(max(1, len(keys)), np.uint64)
    out_o = np.zeros(n + 1, np.int32)
    nnz = ctypes.c_int64()
    st = lib().cvr_truncate_bags(n, offsets.ctypes.data, keys.ctypes.data, max_len, out_o.ctypes.data,
                                 out_k.ctypes.data, ctypes.byref(nnz))
    if st != 0:
        raise CvrError(st, "cvr_truncate_bags")
    return out_k[:nnz.value], out_o


class CvrModel:
    """One libcvr context: model description + workspace + borrowed tables + copied weights.

    ``cfg`` is any object with the fields of ``cvr_synth.CvrConfig`` (n_tables, rows, dim,
    emb_dtype, act_dtype, n_dense, backbone, n_cross, cross_rank, mlp_dims, n_heads, ffn_dim).
    """

    def __init__(self, cfg, max_batch: int, max_nnz: int = 0, world_size: int = 1, rank: int = 0,
                 device: Optional[torch.device] = None, allocate: bool = True, lanes: int = 1):
        self.L = lib()
        self.cfg = cfg
        self._rows = (ctypes.c_int64 * cfg.n_tables)(*cfg.rows)
        self._mlp = (ctypes.c_int * max(1, len(cfg.mlp_dims)))(*cfg.mlp_dims)
        self.desc = cvr_model_desc(
            cfg.n_tables, self._rows, cfg.dim, _DT[cfg.emb_dtype], cfg.n_dense, _DT[cfg.act_dtype],
            _BACKBONE[cfg.backbone], cfg.n_cross, cfg.cross_rank, len(cfg.mlp_dims), self._mlp,
            getattr(cfg, "n_heads", 0), getattr(cfg, "ffn_dim", 0), max_batch, max_nnz, world_size, rank,
            getattr(cfg, "cross_width", 0), getattr(cfg, "n_parallel", 0))
        self.max_batch, self.max_nnz, self.world_size, self.rank = max_batch, max_nnz, world_size, rank
        h = _vp()
        st = self.L.cvr_create(ctypes.byref(self.desc), ctypes.byref(h))
        self.h = h
        if st != 0:
            msg = self.L.cvr_last_error(h).decode() if h.value else ""
            if h.value:
                self.L.cvr_destroy(h)
            self.h = _vp()
            raise CvrError(st, msg)
        self.lanes = lanes
        if lanes != 1:  # executor lanes (cvr.h option "lanes"): before the workspace is sized
            self._check(self.L.cvr_set_option(self.h, b"lanes", lanes))
        ld, dt = ctypes.c_int(), ctypes.c_int()
        self._check(self.L.cvr_x0_layout(self.h, ctypes.byref(ld), ctypes.byref(dt)))
        self.x0_ld, self.x0_dtype = ld.value, {CVR_F32: torch.float32, CVR_BF16: torch.bfloat16}[dt.value]
        n = ctypes.c_size_t()
        self._check(self.L.cvr_workspace_bytes(self.h, ctypes.byref(n)))
        self.workspace_bytes = n.value
        self.workspace = None
        if allocate:
            self.device = torch.device(device or "cuda")
            self.workspace = torch.empty(self.workspace_bytes, dtype=torch.uint8, device=self.device)
            self._check(self.L.cvr_set_workspace(self.h, self.workspace.data_ptr(), self.workspace_bytes))
        self._tables = []

    # -- plumbing ------------------------------------------------------------------------
    def _check(self, st: int):
        if st != 0:
            raise CvrError(st, self.L.cvr_last_error(self.h).decode())

    def close(self):
        if getattr(self, "h", None) is not None and self.h.value:
            self.L.cvr_destroy(self.h)
            self.h = _vp()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- parameters ----------------------------------------------------------------------
    def load_tables(self, tables: Sequence[torch.Tensor], table_ids: Optional[Sequence[int]] = None):
        if table_ids is None:
            table_ids = [t for t in range(self.cfg.n_tables) if t % self.world_size == self.rank]
        n = len(tables)
        ids = (ctypes.c_int * n)(*table_ids)
        ptrs = (_vp * n)(*[t.data_ptr() for t in tables])
        strides = (ctypes.c_int64 * n)(*[t.stride(0) * t.element_size() for t in tables])
        self._check(self.L.cvr_load_tables(self.h, n, ids, ptrs, strides))
        self._tables = list(tables)  # borrowed: keep alive

    def load_weights(self, weights: Dict[str, torch.Tensor]):
        names = list(weights)
        ts = [weights[k].contiguous() for k in names]
        n = len(names)
        cn = (ctypes.c_char_p * n)(*[k.encode() for k in names])
        ptrs = (_vp * n)(*[t.data_ptr() for t in ts])
        dts = (ctypes.c_int * n)(*[_TORCH_DT[t.dtype] for t in ts])
        nd = (ctypes.c_int * n)(*[t.dim() for t in ts])
        flat = [s for t in ts for s in t.shape]
        shp = (ctypes.c_int64 * max(1, len(flat)))(*flat)
        self._check(self.L.cvr_load_weights(self.h, n, cn, ptrs, dts, nd, shp))

    # -- hot path ------------------------------------------------------------------------
    def new_x0(self, batch: int) -> torch.Tensor:
        return torch.empty(batch, self.x0_ld, dtype=self.x0_dtype, device=self.device)

    def embed(self, indices: torch.Tensor, offsets: torch.Tensor, batch: int, dense: Optional[torch.Tensor],
              x0: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
        x0 = self.new_x0(batch) if x0 is None else x0
        self._check(self.L.cvr_embed(self.h, _ptr(indices), _ptr(offsets), indices.numel(), batch, _ptr(dense),
                                     _ptr(x0), _stream(stream)))
        return x0

    def set_feature_spec(self, vocab, pool_mode):
        """cvr_set_feature_spec: per table hash vocab (0 = row ids) and pooling (0 sum, 1 mean)."""
        T = self.cfg.n_tables
        v = (ctypes.c_int64 * T)(*[int(x) for x in vocab])
        pm = (ctypes.c_int * T)(*[int(x) for x in pool_mode])
        self._check(self.L.cvr_set_feature_spec(self.h, T, v, pm))

    def embed_keys(self, keys: torch.Tensor, offsets: torch.Tensor, batch: int, dense: Optional[torch.Tensor],
                   x0: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
        """cvr_embed_keys: keys is an int64 tensor holding the raw 64-bit keys' bit patterns (MISSING = -1)."""
        x0 = self.new_x0(batch) if x0 is None else x0
        self._check(self.L.cvr_embed_keys(self.h, _ptr(keys), _ptr(offsets), keys.numel(), batch, _ptr(dense),
                                          _ptr(x0), _stream(stream)))
        return x0

    def score_keys(self, keys: torch.Tensor, offsets: torch.Tensor, batch: int, dense: Optional[torch.Tensor],
                   scores: Optional[torch.Tensor] = None, s_embed=None, s_dense=None) -> torch.Tensor:
        scores = torch.empty(batch, dtype=torch.float32, device=self.device) if scores is None else scores
        self._check(self.L.cvr_score_keys(self.h, _ptr(keys), _ptr(offsets), keys.numel(), batch, _ptr(dense),
                                          _ptr(scores), _stream(s_embed),
                                          _stream(s_dense if s_dense is not None else s_embed)))
        return scores

    def dense(self, x0: torch.Tensor, batch: int, scores: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
        scores = torch.empty(batch, dtype=torch.float32, device=self.device) if scores is None else scores
        self._check(self.L.cvr_dense(self.h, _ptr(x0), batch, _ptr(scores), _stream(stream)))
        return scores

    def score(self, indices: torch.Tensor, offsets: torch.Tensor, batch: int, dense: Optional[torch.Tensor],
              scores: Optional[torch.Tensor] = None, s_embed=None, s_dense=None) -> torch.Tensor:
        scores = torch.empty(batch, dtype=torch.float32, device=self.device) if scores is None else scores
        self._check(self.L.cvr_score(self.h, _ptr(indices), _ptr(offsets), indices.numel(), batch, _ptr(dense),
                                     _ptr(scores), _stream(s_embed), _stream(s_dense if s_dense is not None else s_embed)))
        return scores

    def score_host(self, indices: torch.Tensor, offsets: torch.Tensor, batch: int, dense: Optional[torch.Tensor],
                   scores: torch.Tensor, s_copy=None, s_embed=None, s_dense=None) -> torch.Tensor:
        """Host-fed S1..S8: CPU (pinned) tensors in, CPU scores out (valid after s_dense syncs)."""
        self._check(self.L.cvr_score_host(self.h, _ptr(indices), _ptr(offsets), indices.numel(), batch, _ptr(dense),
                                          _ptr(scores), _stream(s_copy), _stream(s_embed), _stream(s_dense)))
        return scores

    def warm_graphs(self, max_rows: int, s_embed, s_dense):
        """cvr_warm_graphs: capture every executor graph up to max_rows (nothing runs)."""
        self._check(self.L.cvr_warm_graphs(self.h, max_rows, _stream(s_embed), _stream(s_dense)))

    def status(self, stream=None) -> int:
        """Synchronise ``stream`` and return the sticky device status (raises on CUDA errors)."""
        st = self.L.cvr_get_status(self.h, _stream(stream))
        if st not in (0, CVR_E_INDEX):
            self._check(st)
        return st

    # -- sharded tables -----------------------------------------------------------------------
    def shard_buffer_bytes(self, batch_global: int):
        s, r = ctypes.c_size_t(), ctypes.c_size_t()
        self._check(self.L.cvr_shard_buffer_bytes(self.h, batch_global, ctypes.byref(s), ctypes.byref(r)))
        return s.value, r.value

    def embed_shard(self, indices, offsets, batch_global, dense, send, x0, stream=None):
        self._check(self.L.cvr_embed_shard(self.h, _ptr(indices), _ptr(offsets), indices.numel(), batch_global,
                                           _ptr(dense), _ptr(send), _ptr(x0), _stream(stream)))

    def unpack_shard(self, recv, batch_global, x0, stream=None):
        self._check(self.L.cvr_unpack_shard(self.h, _ptr(recv), batch_global, _ptr(x0), _stream(stream)))

    def set_peers(self, peer_x0_ptrs, peer_ready_ptrs, peer_free_ptrs, local_ready_ptr: int, local_free_ptr: int):
        """peer_x0_ptrs: 2 * N pointers, slot-major ([slot 0 of ranks 0..N-1, slot 1 of ranks 0..N-1])."""
        n = len(peer_ready_ptrs)
        px = (_vp * (2 * n))(*peer_x0_ptrs)
        pr = (_vp * n)(*peer_ready_ptrs)
        pf = (_vp * n)(*peer_free_ptrs)
        self._check(self.L.cvr_set_peers(self.h, n, px, pr, pf, local_ready_ptr, local_free_ptr))

    def embed_fused(self, indices, offsets, batch_global, dense, x0, epoch: int, stream=None):
        self._check(self.L.cvr_embed_fused(self.h, _ptr(indices), _ptr(offsets), indices.numel(), batch_global,
                                           _ptr(dense), _ptr(x0), epoch, _stream(stream)))

    def wait_peers(self, epoch: int, stream=None):
        self._check(self.L.cvr_wait_peers(self.h, epoch, _stream(stream)))

    def release_peers(self, epoch: int, stream=None):
        self._check(self.L.cvr_release_peers(self.h, epoch, _stream(stream)))

    def comm_init(self, unique_id: bytes, world: int, rank: int):
        """cvr_comm_init: the ctx's own NCCL communicator (collective over the ranks)."""
        uid = cvr_nccl_id()
        ctypes.memmove(ctypes.addressof(uid), unique_id, 128)
        self._check(self.L.cvr_comm_init(self.h, ctypes.byref(uid), world, rank))

    def exchange(self, send, recv, batch_global: int, x0, stream=None):
        """cvr_exchange: grouped ncclSend / ncclRecv of the pooled rows + unpack into x0 (S4)."""
        self._check(self.L.cvr_exchange(self.h, _ptr(send), _ptr(recv), batch_global, _ptr(x0), _stream(stream)))

    def executor_slot(self, n: int) -> int:
        """The cvr_call_info slot of the n-th (0-based) executor call: lane n % lanes, that lane's slot."""
        return (n % self.lanes) * EXECUTOR_SLOTS + (n // self.lanes) % EXECUTOR_SLOTS

    def call_info(self, slot: int) -> dict:
        """cvr_call_info: the per-call block of x0 slot `slot` (lane slot // EXECUTOR_SLOTS) as the executor's
        kernels read it; graph_captures counts every lane."""
        rec = cvr_call_record()
        self._check(self.L.cvr_call_info(self.h, slot, ctypes.byref(rec)))
        return {"d_indices": rec.d_indices or 0, "d_keys": rec.d_keys or 0, "d_offsets": rec.d_offsets or 0,
                "d_dense": rec.d_dense or 0, "d_scores": rec.d_scores or 0, "nnz": rec.nnz, "batch": rec.batch,
                "graph_captures": rec.graph_captures}

    def repeat_kernel(self, role: str, reps: int, x0, batch: int, stream=None) -> int:
        """cvr_repeat_kernel: only the GEMMs of `role`, each `reps` times back to back; returns launches."""
        n = ctypes.c_int()
        self._check(self.L.cvr_repeat_kernel(self.h, role.encode(), reps, _ptr(x0), batch, _stream(stream),
                                             ctypes.byref(n)))
        return n.value

    def set_option(self, key: str, value: int):
        self._check(self.L.cvr_set_option(self.h, key.encode(), int(value)))

    def score_raw(self, idx_ptr: int, off_ptr: int, nnz: int, batch: int, dense_ptr: int, scores_ptr: int,
                  s_embed: int, s_dense: int):
        """cvr_score with pre-extracted pointers / stream handles (lowest host overhead)."""
        st = self.L.cvr_score(self.h, idx_ptr, off_ptr, nnz, batch, dense_ptr, scores_ptr, s_embed, s_dense)
        if st:
            self._check(st)

    def score_host_raw(self, idx_ptr: int, off_ptr: int, nnz: int, batch: int, dense_ptr: int, scores_ptr: int,
                       s_copy: int, s_embed: int, s_dense: int):
        st = self.L.cvr_score_host(self.h, idx_ptr, off_ptr, nnz, batch, dense_ptr, scores_ptr, s_copy, s_embed,
                                   s_dense)
        if st:
            self._check(st)

    # -- accounting ----------------------------------------------------------------------------
    def launch_count(self) -> int:
        n = ctypes.c_int64()
        self._check(self.L.cvr_launch_count(self.h, ctypes.byref(n)))
        return n.value

    def profile_begin(self, max_launches: int):
        self._check(self.L.cvr_profile_begin(self.h, max_launches))

    def profile_end(self) -> Dict[str, dict]:
        buf = (cvr_kernel_stat * 32)()
        n = ctypes.c_int()
        self._check(self.L.cvr_profile_end(self.h, buf, 32, ctypes.byref(n)))
        return {buf[i].name.decode(): {"launches": buf[i].launches, "total_ms": buf[i].total_ms,
                                        "avg_ms": buf[i].total_ms / max(1, buf[i].launches),
                                        "min_ms": buf[i].min_ms, "max_ms": buf[i].max_ms}
                for i in range(min(n.value, 16))}
