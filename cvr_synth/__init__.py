"""Seeded synthetic inputs for the CVR scoring hot path (input generator only).

This module is the ONE piece of code shared by the fp64 oracle (``oracle/``) and the
CUDA path (``paper_2605_29232_b200``).  It holds none of the method's arithmetic
(no pooling, no normalisation, no cross / MLP / sigmoid): it only draws the
*inputs* -- embedding-table rows, model parameters, multi-hot bags and raw dense
features -- with the shapes and distributions of ``BASELINE.json`` configs[0..4]
(readings A1-A4, A8, A12, A13, A18-A21 of SURVEY.md §8(c), restated in DESIGN.md §3).

Determinism contract
--------------------
* Table rows are a pure function of (rows seed, table id, row id, column): a
  counter-based splitmix64 hash -> two 24-bit uniforms -> Box-Muller in fp64 ->
  x0.1 (A1: the second argument of N(0, 0.01) is a variance) -> RNE to fp32 ->
  RNE to the storage dtype.  Implemented with torch int64 wrap-around arithmetic so
  the same function runs on CPU (for the oracle's row regeneration) and on a GPU
  (fast materialisation of multi-GB tables).
* Everything else (parameters, bag lengths, indices, dense features, request
  traces) is drawn by numpy ``PCG64`` streams keyed by ``SeedSequence(master,
  spawn_key=(stream, k))``.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from functools import lru_cache
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np
import torch

# ---------------------------------------------------------------------------------
# configurations (BASELINE.json configs[0..4])
# ---------------------------------------------------------------------------------

# exact moments of log1p(10|Z|), Z ~ N(0,1) (pinned by quadrature
# in tests/test_oracle_pins.py::test_norm_constants_quadrature)
NORM_MEAN = 1.940104446397
NORM_STD = 0.764771706179

STREAM_ROWS, STREAM_WEIGHTS, STREAM_LENGTHS, STREAM_INDICES, STREAM_DENSE, STREAM_TRACE = range(6)


@dataclass(frozen=True)
class CvrConfig:
    name: str
    seed: int
    batch: int
    n_tables: int
    rows: Tuple[int, ...]            # rows per table
    dim: int                         # embedding dim d
    emb_dtype: str                   # 'f32' | 'bf16' | 'f16' (table storage)
    act_dtype: str                   # 'f32' | 'bf16' (x0, weights, activations)
    n_dense: int                     # F
    bag: Tuple                       # ('uniform', lo, hi) | ('poisson', lam)
    zipf_a: float
    backbone: str                    # 'dcn_full' | 'dcn_lowrank' | 'ensemble' | 'masknet'
    n_cross: int                     # cross / ensemble layers; masknet: sequential blocks per branch
    cross_rank: int                  # 0 for full rank; masknet: mask hidden width r
    mlp_dims: Tuple[int, ...]        # hidden widths after the backbone (head 1 is implicit)
    n_heads: int = 0                 # ensemble only
    ffn_dim: int = 0                 # ensemble only
    cross_width: int = 0             # masknet: projected cross input width W' (ReLU projection of x0)
    n_parallel: int = 1              # masknet: parallel branches (outputs concatenated)
    scramble: bool = True            # A3
    zipf_mode: str = "truncated"     # A2 ('truncated' | 'clip')

    @property
    def width(self) -> int:
        return self.n_tables * self.dim + self.n_dense

    def with_(self, **kw) -> "CvrConfig":
        d = dict(self.__dict__)
        d.update(kw)
        return CvrConfig(**d)


def _c2_rows(seed: int, n: int) -> Tuple[int, ...]:
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence(seed, spawn_key=(STREAM_ROWS, 1))))
    u = rng.uniform(math.log(1e5), math.log(1e6), size=n)
    return tuple(int(math.floor(math.exp(x))) for x in u)


C1 = CvrConfig("c1", 1001, 256, 8, (1000,) * 8, 16, "f32", "f32", 13, ("uniform", 1, 4), 1.1,
               "dcn_full", 2, 0, (64, 32))
C2 = CvrConfig("c2", 1002, 4096, 26, _c2_rows(1002, 26), 64, "bf16", "bf16", 64, ("poisson", 3.0), 1.05,
               "dcn_lowrank", 3, 256, (1024, 512, 256))
C3 = CvrConfig("c3", 1003, 65536, 100, (10_000_000,) * 100, 128, "f16", "bf16", 64, ("poisson", 5.0), 1.05,
               "dcn_lowrank", 3, 256, (1024, 512, 256))
C3S = C3.with_(name="c3s", seed=1013, rows=(5_000_000,) * 100)
C4 = CvrConfig("c4", 1004, 8192, 64, (1_000_000,) * 64, 256, "bf16", "bf16", 0, ("poisson", 3.0), 1.05,
               "ensemble", 4, 512, (2048, 512), n_heads=4, ffn_dim=1024)
# SURVEY.md §8(f) #1 (not a BASELINE.json config): MaskNet on config 2's features, at the paper's default
# MaskNet scaling factors (Table 1: cross width 2k, deep width 1k, 2 parallel
# blocks, no sequential blocks); mask hidden width r = 512 (unstated; the DCN configs' low-rank reading).
C6 = C2.with_(name="c6", seed=1006, backbone="masknet", n_cross=1, cross_rank=512, cross_width=2048,
              n_parallel=2, mlp_dims=(1024, 512, 256))
CONFIGS: Dict[str, CvrConfig] = {c.name: c for c in (C1, C2, C3, C3S, C4, C6)}  # + C7 (front end) below


# ---------------------------------------------------------------------------------
# dtype helpers (storage rounding is part of the input definition, A13/A14)
# ---------------------------------------------------------------------------------

TORCH_DTYPES = {"f32": torch.float32, "bf16": torch.bfloat16, "f16": torch.float16}


def round_to(x64: torch.Tensor, dtype: str) -> torch.Tensor:
    """RNE fp64 -> fp32 -> storage dtype (the stored value *is* the model, A13)."""
    return x64.to(torch.float32).to(TORCH_DTYPES[dtype])


# ---------------------------------------------------------------------------------
# counter-based table rows
# ---------------------------------------------------------------------------------

_GOLDEN = 0x9E3779B97F4A7C15 - (1 << 64)
_M1 = 0xBF58476D1CE4E5B9 - (1 << 64)
_M2 = 0x94D049BB133111EB - (1 << 64)


def _srl(x: torch.Tensor, s: int) -> torch.Tensor:
    """Logical right shift of int64 viewed as uint64."""
    return (x >> s) & ((1 << (64 - s)) - 1)


def splitmix64(x: torch.Tensor) -> torch.Tensor:
    """splitmix64 output function on int64 (uint64 semantics via wrap-around)."""
    z = x
    z = (z ^ _srl(z, 30)) * _M1
    z = (z ^ _srl(z, 27)) * _M2
    return z ^ _srl(z, 31)


def _s64(v: int) -> int:
    v &= (1 << 64) - 1
    return v - (1 << 64) if v >= (1 << 63) else v


def rows_seed(cfg: CvrConfig) -> int:
    ss = np.random.SeedSequence(cfg.seed, spawn_key=(STREAM_ROWS,))
    return int(ss.generate_state(1, np.uint64)[0])


def table_rows(seed: int, t: int, row_ids: torch.Tensor, d: int, dtype: str) -> torch.Tensor:
    """Rows ``row_ids`` of table ``t``: [n, d] in storage dtype, on row_ids.device.

    counter(t, r, p) = t<<40 | r<<8 | p for column pair p = c//2 (d <= 512, rows < 2^32);
    z = splitmix64(seed + (counter+1)*golden); u1 = (z>>>40 + 1)/2^24 in (0,1],
    u2 = ((z>>>16) & (2^24-1))/2^24; n0 = sqrt(-2 ln u1) cos(2 pi u2), n1 = ... sin.
    """
    assert d % 2 == 0 and d <= 512
    dev = row_ids.device
    r = row_ids.to(torch.int64).reshape(-1, 1)
    p = torch.arange(d // 2, device=dev, dtype=torch.int64).reshape(1, -1)
    ctr = (int(t) << 40) | (r << 8) | p
    z = splitmix64(_s64(seed) + (ctr + 1) * _GOLDEN)
    u1 = (_srl(z, 40) + 1).to(torch.float64) * (2.0 ** -24)
    u2 = (_srl(z, 16) & 0xFFFFFF).to(torch.float64) * (2.0 ** -24)
    rad = torch.sqrt(-2.0 * torch.log(u1))
    ang = (2.0 * math.pi) * u2
    out = torch.empty(r.shape[0], d // 2, 2, dtype=torch.float64, device=dev)
    out[:, :, 0] = rad * torch.cos(ang)
    out[:, :, 1] = rad * torch.sin(ang)
    return round_to(0.1 * out.reshape(r.shape[0], d), dtype)


class TableSpec:
    """Lazy handle on one embedding table: regenerate any rows on demand."""

    def __init__(self, seed: int, t: int, n_rows: int, d: int, dtype: str):
        self.seed, self.t, self.n_rows, self.d, self.dtype = seed, t, n_rows, d, dtype

    def gather(self, row_ids, device="cpu") -> torch.Tensor:
        ids = torch.as_tensor(np.asarray(row_ids, dtype=np.int64), device=device)
        return table_rows(self.seed, self.t, ids, self.d, self.dtype)

    def gather_f64(self, row_ids) -> np.ndarray:
        """Stored values widened exactly to fp64 (numpy) -- what the oracle consumes."""
        return self.gather(row_ids).to(torch.float64).numpy()

    def materialize(self, device="cpu", chunk_rows: int = 1 << 20) -> torch.Tensor:
        out = torch.empty(self.n_rows, self.d, dtype=TORCH_DTYPES[self.dtype], device=device)
        for s in range(0, self.n_rows, chunk_rows):
            e = min(self.n_rows, s + chunk_rows)
            out[s:e] = table_rows(self.seed, self.t, torch.arange(s, e, device=device), self.d, self.dtype)
        return out


def table_specs(cfg: CvrConfig) -> List[TableSpec]:
    seed = rows_seed(cfg)
    return [TableSpec(seed, t, cfg.rows[t], cfg.dim, cfg.emb_dtype) for t in range(cfg.n_tables)]


# ---------------------------------------------------------------------------------
# parameters (A1, A12, A13)
# ---------------------------------------------------------------------------------

def weight_shapes(cfg: CvrConfig) -> List[Tuple[str, Tuple[int, ...]]]:
    """Names and [out, in] shapes of every parameter, in draw order."""
    W = cfg.width
    s: List[Tuple[str, Tuple[int, ...]]] = []
    if cfg.n_dense:
        s += [("norm/mean", (cfg.n_dense,)), ("norm/std", (cfg.n_dense,))]
    if cfg.backbone == "dcn_full":
        for l in range(cfg.n_cross):
            s += [(f"dcn/{l}/W", (W, W)), (f"dcn/{l}/b", (W,))]
        prev = W
    elif cfg.backbone == "dcn_lowrank":
        for l in range(cfg.n_cross):
            s += [(f"dcn/{l}/V", (cfg.cross_rank, W)), (f"dcn/{l}/U", (W, cfg.cross_rank)), (f"dcn/{l}/b", (W,))]
        prev = W
    elif cfg.backbone == "ensemble":
        D = cfg.dim
        for l in range(cfg.n_cross):
            s += [(f"ens/{l}/dcn/V", (cfg.cross_rank, W)), (f"ens/{l}/dcn/U", (W, cfg.cross_rank)),
                  (f"ens/{l}/dcn/b", (W,)),
                  (f"ens/{l}/mha/Wqkv", (3 * D, D)), (f"ens/{l}/mha/bqkv", (3 * D,)),
                  (f"ens/{l}/mha/Wo", (D, D)), (f"ens/{l}/mha/bo", (D,)),
                  (f"ens/{l}/ffn/W1", (cfg.ffn_dim, D)), (f"ens/{l}/ffn/b1", (cfg.ffn_dim,)),
                  (f"ens/{l}/ffn/W2", (D, cfg.ffn_dim)), (f"ens/{l}/ffn/b2", (D,)),
                  (f"ens/{l}/ln/gamma", (D,)), (f"ens/{l}/ln/beta", (D,))]
        prev = W
    elif cfg.backbone == "masknet":
        Wp = cfg.cross_width or W
        if cfg.cross_width:
            s += [("proj/W", (Wp, W)), ("proj/b", (Wp,))]
        for p in range(cfg.n_parallel):
            for q in range(cfg.n_cross):
                s += [(f"mask/{p}/{q}/V", (cfg.cross_rank, Wp)), (f"mask/{p}/{q}/c", (cfg.cross_rank,)),
                      (f"mask/{p}/{q}/U", (Wp, cfg.cross_rank)), (f"mask/{p}/{q}/b", (Wp,))]
        prev = cfg.n_parallel * Wp
    else:
        raise ValueError(cfg.backbone)
    for i, h in enumerate(cfg.mlp_dims):
        s += [(f"mlp/{i}/W", (h, prev)), (f"mlp/{i}/b", (h,))]
        prev = h
    s += [("head/w", (1, prev)), ("head/b", (1,))]
    return s


def make_weights(cfg: CvrConfig) -> Dict[str, torch.Tensor]:
    """All parameters as CPU tensors in the act dtype (norm stats always fp32)."""
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence(cfg.seed, spawn_key=(STREAM_WEIGHTS,))))
    out: Dict[str, torch.Tensor] = {}
    for name, shape in weight_shapes(cfg):
        role = name.rsplit("/", 1)[-1]
        if name == "norm/mean":
            x = np.full(shape, NORM_MEAN)
        elif name == "norm/std":
            x = np.full(shape, NORM_STD)
        elif role == "gamma" or (name.startswith("mask/") and role == "b"):
            # multiplicative parameters start around 1 (A12 for LN gamma; A27 for the MaskNet mask bias)
            x = 1.0 + rng.normal(0.0, 0.1, size=shape)
        elif len(shape) == 1 or role in ("beta",):
            x = rng.normal(0.0, 0.1, size=shape)          # biases: N(0, 0.01) (variance), A12
        else:
            fan_in = shape[1]
            x = rng.normal(0.0, 1.0 / math.sqrt(fan_in), size=shape)   # N(0, 1/fan_in), A1/A12
        dt = "f32" if name.startswith("norm/") else cfg.act_dtype
        out[name] = round_to(torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)), dt)
    return out


# ---------------------------------------------------------------------------------
# indices: truncated Zipf (A2) + scramble (A3)
# ---------------------------------------------------------------------------------

@lru_cache(maxsize=64)
def _zipf_cdf(n: int, a: float) -> np.ndarray:
    k = np.arange(1, n + 1, dtype=np.float64)
    c = np.cumsum(k ** (-a))
    return c / c[-1]


@lru_cache(maxsize=256)
def scramble_multiplier(n: int) -> int:
    """A3: P = 2654435761 mod N, incremented until gcd(P, N) = 1 and P not in {0, 1}."""
    p = 2654435761 % n
    while p in (0, 1) or math.gcd(p, n) != 1:
        p += 1
        if p >= n:
            p = 2
    return p


def sample_zipf_rows(rng: np.random.Generator, n_rows: int, a: float, size: int,
                     scramble: bool = True, mode: str = "truncated") -> np.ndarray:
    if mode == "truncated":
        cdf = _zipf_cdf(n_rows, a)
        k = np.searchsorted(cdf, rng.random(size), side="right") + 1   # rank in 1..N
        k = np.minimum(k, n_rows)
    elif mode == "clip":
        k = np.minimum(rng.zipf(a, size), n_rows)
    elif mode == "uniform":
        k = rng.integers(1, n_rows + 1, size)
    else:
        raise ValueError(mode)
    r = k.astype(np.int64) - 1
    if scramble and n_rows > 2:
        r = (r * scramble_multiplier(n_rows)) % n_rows
    return r


def _rng(cfg: CvrConfig, stream: int, k: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence(cfg.seed, spawn_key=(stream, k))))


@dataclass
class Batch:
    """One batch of inputs in the library's layout (SURVEY.md §8(b) input conventions).

    offsets: int32 [T*B+1], table-major: bag (t, b) = indices[offsets[t*B+b]:offsets[t*B+b+1]]
    indices: int32 [nnz], per-table local row ids
    dense:   fp32  [B, F] raw log1p values
    """
    batch: int
    n_tables: int
    indices: np.ndarray
    offsets: np.ndarray
    dense: np.ndarray
    lengths: np.ndarray = field(repr=False, default=None)

    @property
    def nnz(self) -> int:
        return int(self.offsets[-1])


def sub_batch(bt: Batch, sel) -> Batch:
    """Examples ``sel`` of ``bt`` as their own batch (same bags, same order): CSR slicing only."""
    sel = np.asarray(sel)
    T, B = bt.n_tables, bt.batch
    idx, off = [], [0]
    for t in range(T):
        for b in sel:
            seg = bt.indices[bt.offsets[t * B + b]:bt.offsets[t * B + b + 1]]
            idx.append(seg)
            off.append(off[-1] + len(seg))
    idx = np.concatenate(idx) if idx else np.zeros(0, np.int32)
    return Batch(len(sel), T, idx.astype(np.int32), np.array(off, np.int32), bt.dense[sel])


def bag_lengths(cfg: CvrConfig, k: int, batch: Optional[int] = None) -> np.ndarray:
    B = cfg.batch if batch is None else batch
    rng = _rng(cfg, STREAM_LENGTHS, k)
    kind = cfg.bag[0]
    if kind == "uniform":
        L = rng.integers(cfg.bag[1], cfg.bag[2] + 1, size=(cfg.n_tables, B))
    elif kind == "poisson":
        L = rng.poisson(cfg.bag[1], size=(cfg.n_tables, B)) + 1
    else:
        raise ValueError(kind)
    return L.astype(np.int64)


def make_batch(cfg: CvrConfig, k: int, batch: Optional[int] = None, tables: Optional[Sequence[int]] = None,
               index_mode: Optional[str] = None) -> Batch:
    """Batch number k of config cfg (seeded).  ``tables`` restricts to a subset of tables
    (sharded mode: the local tables over the global batch), keeping per-table draws
    identical to the unsharded batch."""
    B = cfg.batch if batch is None else batch
    L = bag_lengths(cfg, k, B)
    tl = list(range(cfg.n_tables)) if tables is None else list(tables)
    idx_parts = []
    mode = index_mode or cfg.zipf_mode
    for t in tl:
        rng = _rng(cfg, STREAM_INDICES, k * 4096 + t)
        idx_parts.append(sample_zipf_rows(rng, cfg.rows[t], cfg.zipf_a, int(L[t].sum()), cfg.scramble, mode))
    Ls = L[tl]
    offsets = np.zeros(len(tl) * B + 1, dtype=np.int64)
    offsets[1:] = np.cumsum(Ls.reshape(-1))
    indices = np.concatenate(idx_parts) if idx_parts else np.zeros(0, np.int64)
    rng = _rng(cfg, STREAM_DENSE, k)
    dense = np.log1p(np.abs(rng.normal(size=(B, cfg.n_dense))) * 10.0).astype(np.float32)
    return Batch(B, len(tl), indices.astype(np.int32), offsets.astype(np.int32), dense, Ls)


# ---------------------------------------------------------------------------------
# feature front end: raw categorical keys, text strings, item histories
# ---------------------------------------------------------------------------------
# config c7 = config 2's model on raw features: tables 0..19 categorical (multi-hot 64-bit keys, 1% MISSING,
# sum), 20..22 text (character 3-grams of 1-4 word queries, 2% empty, mean), 23..25 item histories
# (Poisson(30) keys, 10% long Poisson(120), truncated to the 50 most recent, mean); every table hashed with
# vocab = rows - 1 (the last row is the `unseen' row).  Readings A28 (MISSING key), A29 (byte n-grams).
C7 = C2.with_(name="c7", seed=1007)
FRONTEND_C7 = {"kinds": ["cat"] * 20 + ["text"] * 3 + ["seq"] * 3, "ngram": 3, "max_len": 50, "missing": 0.01}
STREAM_FRONTEND = 11
KEY_MISSING_U64 = np.uint64(0xFFFFFFFFFFFFFFFF)


CONFIGS["c7"] = C7


def _mix64(x: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser (a PRNG step of the generator, not the method's hash): ranks -> 64-bit ids."""
    z = x.astype(np.uint64) + np.uint64(0x9E3779B97F4A7C15)
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


@dataclass
class FeatureBatch:
    """Raw features of one batch: per table either ('keys', keys uint64 [n], offsets int32 [B+1]) for
    categorical / sequential tables (histories oldest first), or ('text', [bytes] * B)."""
    batch: int
    tables: List[Tuple]
    dense: np.ndarray


def make_feature_batch(cfg: CvrConfig, k: int, batch: Optional[int] = None, spec=FRONTEND_C7) -> FeatureBatch:
    B = cfg.batch if batch is None else batch
    rng = _rng(cfg, STREAM_FRONTEND, k)
    words = None
    out = []
    for t, kind in enumerate(spec["kinds"]):
        if kind in ("cat", "seq"):
            if kind == "cat":
                L = rng.poisson(3.0, size=B) + 1
            else:
                long = rng.random(B) < 0.1
                L = np.where(long, rng.poisson(120.0, size=B), rng.poisson(30.0, size=B))
            n = int(L.sum())
            ranks = sample_zipf_rows(rng, 10 * cfg.rows[t], cfg.zipf_a, n, scramble=False)
            keys = _mix64(ranks.astype(np.uint64) * np.uint64(4096) + np.uint64(t))
            if kind == "cat":
                keys[rng.random(n) < spec["missing"]] = KEY_MISSING_U64
            off = np.zeros(B + 1, np.int32)
            off[1:] = np.cumsum(L)
            out.append(("keys", keys, off))
        else:
            if words is None:
                wl = rng.integers(3, 10, size=5000)
                letters = rng.integers(97, 123, size=int(wl.sum()))
                pos = np.concatenate([[0], np.cumsum(wl)])
                words = [bytes(letters[pos[i]:pos[i + 1]].astype(np.uint8)) for i in range(5000)]
            texts = []
            for b in range(B):
                if rng.random() < 0.02:
                    texts.append(b"")
                    continue
                nw = int(rng.integers(1, 5))
                ids = sample_zipf_rows(rng, 5000, 1.1, nw, scramble=False)
                texts.append(b" ".join(words[i] for i in ids))
            out.append(("text", texts))
    rngd = _rng(cfg, STREAM_DENSE, 10_000 + k)
    dense = np.log1p(np.abs(rngd.normal(size=(B, cfg.n_dense))) * 10.0).astype(np.float32)
    return FeatureBatch(B, out, dense)


# ---------------------------------------------------------------------------------
# serving traces (config 5, A21)
# ---------------------------------------------------------------------------------

def request_trace(qps: float, duration_s: float, seed: int = 1005, mu: float = math.log(50.0),
                  sigma: float = 0.8, cap: int = 500) -> Tuple[np.ndarray, np.ndarray]:
    """Open-loop Poisson arrivals: (scheduled arrival times [s], items per request)."""
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence(seed, spawn_key=(STREAM_TRACE, int(qps)))))
    n_est = int(qps * duration_s * 1.2) + 16
    gaps = rng.exponential(1.0 / qps, size=n_est)
    t = np.cumsum(gaps)
    while t[-1] < duration_s:
        t = np.concatenate([t, t[-1] + np.cumsum(rng.exponential(1.0 / qps, size=n_est))])
    t = t[t < duration_s]
    n = np.clip(np.rint(np.exp(mu + sigma * rng.normal(size=t.shape[0]))), 1, cap).astype(np.int64)
    return t, n


def make_item_pool(cfg: CvrConfig, pool_size: int = 1 << 16, k: int = 5000) -> Batch:
    """A seeded pool of config-style items (A21: items draw from a seeded pool): the features of
    ``pool_size`` candidate items as one batch (table-major CSR + dense rows)."""
    return make_batch(cfg, k, batch=pool_size)


def make_requests_flat(qps: float, duration_s: float, pool_size: int, seed: int = 1005):
    """Config 5 trace as flat arrays for the native serving loop (large offered loads): (t_arrival [s], n_items,
    item_start [n+1], item_ids) -- the same arrivals and sizes as make_requests, item ids drawn in one call."""
    t, n = request_trace(qps, duration_s, seed=seed)
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence(seed, spawn_key=(STREAM_TRACE, 8, int(qps)))))
    start = np.zeros(len(n) + 1, np.int64)
    start[1:] = np.cumsum(n)
    return t, n.astype(np.int32), start, rng.integers(0, pool_size, int(start[-1])).astype(np.int32)


def make_requests(qps: float, duration_s: float, pool_size: int, seed: int = 1005):
    """Config 5 request trace: [(t_arrival, item_ids)], Poisson arrivals at ``qps`` queries/s, items per
    query clip(rint(lognormal(ln 50, 0.8)), 1, 500) drawn uniformly from the pool (A21)."""
    t, n = request_trace(qps, duration_s, seed=seed)
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence(seed, spawn_key=(STREAM_TRACE, 7, int(qps)))))
    return [(float(ti), rng.integers(0, pool_size, int(ni)).astype(np.int32)) for ti, ni in zip(t, n)]
