"""fp64 CPU oracle for the CVR scoring hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_2605_29232_b200``) never imports it, and it never imports the product path:
the two share no code, only the seeded input generator ``cvr_synth`` (which holds no
arithmetic of the method).

Every function is the plain definition of one step, evaluated in numpy float64
(PAPER.md = /root/reference/PAPER.md, the paper's LaTeX source; SURVEY.md §8(c) gives
the readings A1..A26 used where the paper is silent, restated in DESIGN.md §3):

  O2 pool       p[b,t,:] = sum_{j in bag(t,b)} E_t[idx_j, :]      PAPER.md:96 (§2.1 "Each
                categorical feature is designated to an embedding layer"); north star (a)
  O3 normalize  z = (x - mu) / sigma                                PAPER.md:95 (§2.1), A8
  O4 concat     x0 = [p_0 | ... | p_{T-1} | z]                      PAPER.md:227 (x_0), A7
  O5 cross      full:     x_{l+1} = x0 * (W_l x_l + b_l) + x_l      PAPER.md:116-119 (eq:dcnv2)
                low rank: x_{l+1} = x0 * (U_l (V_l x_l) + b_l) + x_l  PAPER.md:225 (§3.1), A9
  O6 MLP        h_{i+1} = max(0, M_i h_i + c_i)                     PAPER.md:229-233, A10/A11
  O7 head       s = sigmoid(m . h + c)                              BASELINE.json north star, A16
  O8 ensemble   Y = LN_token(DCN(X) + MHA(X) + FFN(X))              PAPER.md:243-258, A20
                (the paper gives no formula for the ensemble layer: pinned to the A20 reading by the
                 hand-derived goldens E8 -- two-head attention with 1/sqrt(dh) != 1/dh, non-uniform
                 softmax, per-token queries; FFN with live ReLU and b2; a layer with X0 != X_l --
                 P16, and P8 scalar brute force, tests/test_oracle_pins.py)
  O10 MaskNet   x0' = ReLU(W_in x0 + b_in)                         PAPER.md:227-228 ("scale the
                input x0 via one-layer relu projection"); block
                x_{l+1} = (U_l ReLU(V_l x0' + c_l) + b_l) * x_l      PAPER.md:226 (eq. "MaskNet uses"),
                no residual; parallel branches concatenated / sequential
                blocks chained; biases c_l, b_l per reading A27
  O11 front end hashed keys -> rows: FNV-1a 64 over the key's 8 big-endian bytes mod vocab,
                MISSING -> the `unseen' row vocab ("hashing trick", PAPER.md:287
                "a unique `unseen' placeholder"); text -> character n-gram
                keys, mean pooled; sequences truncated to the most recent max_len
                keys, mean pooled; empty bag -> 0

Parameters are the *stored* (fp32 / bf16 / fp16) values widened exactly to fp64 (A13).
"""
from __future__ import annotations

import math
from typing import Dict, List, Sequence

import numpy as np

__all__ = [
    "validate_csr", "embedding_bag_sum", "normalize_dense", "concat_x0", "cross_full",
    "cross_lowrank", "mlp_relu", "head_logit", "sigmoid", "layer_norm_tokens", "mha_tokens",
    "ffn_tokens", "ensemble_layer", "masknet_project", "masknet_block", "masknet_forward", "score_forward",
    "dense_forward", "to_f64", "fnv1a64", "hash_index", "KEY_MISSING", "ngram_keys", "truncate_recent",
    "embedding_bag", "frontend_rows",
]


class OracleInputError(ValueError):
    """Malformed CSR or out-of-range index (the GPU path reports CVR_E_INDEX), A23."""


def to_f64(x) -> np.ndarray:
    """Widen a stored parameter / table (torch or numpy) exactly to fp64."""
    if hasattr(x, "detach"):
        import torch
        return x.detach().to("cpu", torch.float64).numpy()
    return np.asarray(x, dtype=np.float64)


# -- O1 ---------------------------------------------------------------------------------
def validate_csr(indices: np.ndarray, offsets: np.ndarray, rows: Sequence[int], n_tables: int, batch: int) -> None:
    """A23: offsets[0] = 0, non-decreasing, offsets[T*B] = nnz, 0 <= idx < rows_t."""
    offsets = np.asarray(offsets, dtype=np.int64)
    indices = np.asarray(indices, dtype=np.int64)
    if offsets.shape != (n_tables * batch + 1,):
        raise OracleInputError(f"offsets shape {offsets.shape} != ({n_tables * batch + 1},)")
    if offsets[0] != 0 or np.any(np.diff(offsets) < 0) or offsets[-1] != indices.shape[0]:
        raise OracleInputError("offsets not a valid CSR row pointer")
    for t in range(n_tables):
        seg = indices[offsets[t * batch]:offsets[(t + 1) * batch]]
        if seg.size and (seg.min() < 0 or seg.max() >= rows[t]):
            raise OracleInputError(f"table {t}: index out of range [0, {rows[t]})")


# -- O2 ---------------------------------------------------------------------------------
def embedding_bag_sum(tables: Sequence, indices: np.ndarray, offsets: np.ndarray, n_tables: int,
                      batch: int, dim: int) -> np.ndarray:
    """O2 (north star (a) "sum-pool"): p[b, t, :] = sum of the bag's rows,
    duplicates counted with multiplicity (A5), empty bag -> 0 (A4).

    ``tables[t]`` is an fp64 array [rows_t, d] or an object with ``gather_f64(ids)``.
    Summation is in index order (np.add.at is unbuffered and sequential).
    """
    indices = np.asarray(indices, dtype=np.int64)
    offsets = np.asarray(offsets, dtype=np.int64)
    p = np.zeros((n_tables, batch, dim), dtype=np.float64)
    for t in range(n_tables):
        lo, hi = offsets[t * batch], offsets[(t + 1) * batch]
        ids = indices[lo:hi]
        tab = tables[t]
        rows = tab.gather_f64(ids) if hasattr(tab, "gather_f64") else np.asarray(tab, np.float64)[ids]
        lens = np.diff(offsets[t * batch:(t + 1) * batch + 1])
        bag_of = np.repeat(np.arange(batch), lens)
        np.add.at(p[t], bag_of, rows)
    return p.transpose(1, 0, 2)  # [B, T, d]


def embedding_bag(tables: Sequence, indices: np.ndarray, offsets: np.ndarray, n_tables: int, batch: int, dim: int,
                  modes: Sequence[str]) -> np.ndarray:
    """O2 / O11: per-table pooling mode 'sum' (north star (a)) or 'mean' ("average pooling";
    SPEC.md:169-186): mean = sum / bag length; an empty bag pools to 0 in both modes."""
    p = embedding_bag_sum(tables, indices, offsets, n_tables, batch, dim)
    offsets = np.asarray(offsets, dtype=np.int64)
    for t in range(n_tables):
        if modes[t] == "mean":
            L = np.diff(offsets[t * batch:(t + 1) * batch + 1]).astype(np.float64)
            p[:, t, :] /= np.maximum(L, 1.0)[:, None]
        elif modes[t] != "sum":
            raise ValueError(modes[t])
    return p


# -- O11 feature front end ----------------------------------------------------------------
KEY_MISSING = (1 << 64) - 1   # reading A28: the MISSING categorical value -> the unseen row
_FNV_OFFSET, _FNV_PRIME, _M64 = 0xCBF29CE484222325, 0x100000001B3, (1 << 64) - 1


def fnv1a64(data: bytes) -> int:
    """FNV-1a, 64 bit: h = offset basis; for each byte: h ^= byte; h *= prime (mod 2^64)."""
    h = _FNV_OFFSET
    for byte in data:
        h ^= byte
        h = (h * _FNV_PRIME) & _M64
    return h


def hash_index(key: int, vocab: int) -> int:
    """FNV-1a 64 over the key's 8 big-endian bytes, modulo vocab; KEY_MISSING -> vocab
    (the appended `unseen' row)."""
    if vocab < 1:
        raise ValueError("vocab_size >= 1")
    if int(key) == KEY_MISSING:
        return vocab
    return fnv1a64(int(key).to_bytes(8, "big")) % vocab


def ngram_keys(text: bytes, n: int) -> List[int]:
    """PAPER.md:97 "tokenized into character n-grams": the overlapping n-byte grams of ``text`` (reading A29:
    bytes), each packed big-endian into a 64-bit key (n <= 8), in order; fewer than n bytes -> no grams."""
    if not 1 <= n <= 8:
        raise ValueError("1 <= n <= 8")
    return [int.from_bytes(text[i:i + n], "big") for i in range(len(text) - n + 1)]


def truncate_recent(keys: Sequence[int], max_len: int) -> List[int]:
    """keep the most recent max_len keys of a history (oldest first, most recent last)."""
    keys = list(keys)
    return keys[len(keys) - max_len:] if len(keys) > max_len else keys


# -- O3 / O4 ----------------------------------------------------------------------------
def normalize_dense(x: np.ndarray, mean: np.ndarray, std: np.ndarray) -> np.ndarray:
    """O3 ("normal standardization"; A8): z = (x - mu) / max(sigma, 1e-8)."""
    return (np.asarray(x, np.float64) - to_f64(mean)) / np.maximum(to_f64(std), 1e-8)


def concat_x0(pooled: np.ndarray, z: np.ndarray) -> np.ndarray:
    """O4 (A7): x0 = [p_0 | ... | p_{T-1} | z], tables in id order, then dense features."""
    B = pooled.shape[0]
    return np.concatenate([pooled.reshape(B, -1), z.reshape(B, -1)], axis=1)


# -- O5 ---------------------------------------------------------------------------------
def cross_full(x0: np.ndarray, xl: np.ndarray, W: np.ndarray, b: np.ndarray) -> np.ndarray:
    """O5 full rank (eq:dcnv2): x_{l+1} = x0 * (W x_l + b) + x_l.
    Row-vector form: rows of xl are examples, W is [out, in]."""
    return x0 * (xl @ W.T + b) + xl


def cross_lowrank(x0: np.ndarray, xl: np.ndarray, U: np.ndarray, V: np.ndarray, b: np.ndarray) -> np.ndarray:
    """O5 low rank (A9): x_{l+1} = x0 * (U (V x_l) + b) + x_l; V [r, W], U [W, r]."""
    return x0 * ((xl @ V.T) @ U.T + b) + xl


# -- O6 / O7 ----------------------------------------------------------------------------
def mlp_relu(h: np.ndarray, M: np.ndarray, c: np.ndarray) -> np.ndarray:
    """O6 (A11): h' = max(0, M h + c), M [out, in]."""
    return np.maximum(h @ M.T + c, 0.0)


def head_logit(h: np.ndarray, m: np.ndarray, c: np.ndarray) -> np.ndarray:
    """O7: z = m . h + c (m [1, in])."""
    return h @ np.asarray(m).reshape(-1) + np.asarray(c).reshape(-1)[0]


def sigmoid(z: np.ndarray) -> np.ndarray:
    """O7 / A16: numerically stable two-branch logistic."""
    z = np.asarray(z, np.float64)
    out = np.empty_like(z)
    pos = z >= 0
    out[pos] = 1.0 / (1.0 + np.exp(-z[pos]))
    ez = np.exp(z[~pos])
    out[~pos] = ez / (1.0 + ez)
    return out


# -- O8 (config 4, A20) -----------------------------------------------------------------
def layer_norm_tokens(y: np.ndarray, gamma: np.ndarray, beta: np.ndarray, eps: float = 1e-5) -> np.ndarray:
    """Per-token LayerNorm over the last axis, biased variance (A20)."""
    mu = y.mean(axis=-1, keepdims=True)
    var = ((y - mu) ** 2).mean(axis=-1, keepdims=True)
    return (y - mu) / np.sqrt(var + eps) * gamma + beta


def mha_tokens(X: np.ndarray, Wqkv: np.ndarray, bqkv: np.ndarray, Wo: np.ndarray, bo: np.ndarray,
               n_heads: int) -> np.ndarray:
    """Multi-head self-attention over the S tokens of each example (A20):
    Q,K,V = X W^T + b; per head softmax(Q K^T / sqrt(dh)) V; output W_o concat + b_o."""
    B, S, D = X.shape
    dh = D // n_heads
    qkv = X @ Wqkv.T + bqkv                                   # [B, S, 3D]
    q, k, v = qkv[..., :D], qkv[..., D:2 * D], qkv[..., 2 * D:]
    q = q.reshape(B, S, n_heads, dh).transpose(0, 2, 1, 3)
    k = k.reshape(B, S, n_heads, dh).transpose(0, 2, 1, 3)
    v = v.reshape(B, S, n_heads, dh).transpose(0, 2, 1, 3)
    s = q @ k.transpose(0, 1, 3, 2) / math.sqrt(dh)           # [B, H, S, S]
    s = s - s.max(axis=-1, keepdims=True)
    p = np.exp(s)
    p = p / p.sum(axis=-1, keepdims=True)
    o = (p @ v).transpose(0, 2, 1, 3).reshape(B, S, D)
    return o @ Wo.T + bo


def ffn_tokens(X: np.ndarray, W1: np.ndarray, b1: np.ndarray, W2: np.ndarray, b2: np.ndarray) -> np.ndarray:
    """Per-token FFN W2 ReLU(W1 x + b1) + b2 (A20)."""
    return np.maximum(X @ W1.T + b1, 0.0) @ W2.T + b2


def ensemble_layer(X0: np.ndarray, Xl: np.ndarray, P: Dict[str, np.ndarray], l: int, n_heads: int,
                   n_tokens: int) -> np.ndarray:
    """O8 (A20): Y = LN_token(DCN(X) + MHA(X) + FFN(X)); DCN acts on the flattened vector
    with x0 = the layer-0 input.  X0, Xl: [B, S*D]."""
    B = Xl.shape[0]
    g = lambda n: P[f"ens/{l}/{n}"]
    dcn = cross_lowrank(X0, Xl, g("dcn/U"), g("dcn/V"), g("dcn/b"))
    Xt = Xl.reshape(B, n_tokens, -1)
    mha = mha_tokens(Xt, g("mha/Wqkv"), g("mha/bqkv"), g("mha/Wo"), g("mha/bo"), n_heads)
    ffn = ffn_tokens(Xt, g("ffn/W1"), g("ffn/b1"), g("ffn/W2"), g("ffn/b2"))
    y = dcn.reshape(B, n_tokens, -1) + mha + ffn
    return layer_norm_tokens(y, g("ln/gamma"), g("ln/beta")).reshape(B, -1)


# -- O10 MaskNet ----------------------------------------------------
def masknet_project(x0: np.ndarray, W: np.ndarray, b: np.ndarray) -> np.ndarray:
    """"scale the input x0 via one-layer relu projection": x0' = max(0, W x0 + b),
    W [W', W] (the cross width W' of Table 1)."""
    return np.maximum(x0 @ W.T + b, 0.0)


def masknet_block(x_in: np.ndarray, x0p: np.ndarray, U: np.ndarray, V: np.ndarray, c: np.ndarray,
                  b: np.ndarray) -> np.ndarray:
    """x_{l+1} = U_l(ReLU(V_l x0)) * x_l, biases per A27: (U ReLU(V x0' + c) + b) * x_in.
    No residual ("omits the residual connection present in DCNv2").  V [r, W'], U [W', r]."""
    return (np.maximum(x0p @ V.T + c, 0.0) @ U.T + b) * x_in


def masknet_forward(cfg, P: Dict[str, np.ndarray], x0: np.ndarray) -> np.ndarray:
    """n_parallel branches, each a chain of n_cross blocks M(x, x0') starting from x0',
    concatenated in branch order ("Concat(M_0(x0, x0), ...)" / "M_n(...M_1(x0, x0)..., x0)"; SPEC.md's
    mixed mode = a sequential chain inside each parallel branch)."""
    x0p = masknet_project(x0, P["proj/W"], P["proj/b"]) if cfg.cross_width else x0
    outs = []
    for p in range(cfg.n_parallel):
        x = x0p
        for q in range(cfg.n_cross):
            g = lambda n: P[f"mask/{p}/{q}/{n}"]
            x = masknet_block(x, x0p, g("U"), g("V"), g("c"), g("b"))
        outs.append(x)
    return np.concatenate(outs, axis=1)


# -- whole path -------------------------------------------------------------------------
def dense_forward(cfg, P: Dict[str, np.ndarray], x0: np.ndarray) -> Dict[str, np.ndarray]:
    """S5-S7 on an fp64 x0 [B, W]: backbone, MLP tower, head, sigmoid."""
    xl = x0
    if cfg.backbone == "dcn_full":
        for l in range(cfg.n_cross):
            xl = cross_full(x0, xl, P[f"dcn/{l}/W"], P[f"dcn/{l}/b"])
    elif cfg.backbone == "dcn_lowrank":
        for l in range(cfg.n_cross):
            xl = cross_lowrank(x0, xl, P[f"dcn/{l}/U"], P[f"dcn/{l}/V"], P[f"dcn/{l}/b"])
    elif cfg.backbone == "ensemble":
        for l in range(cfg.n_cross):
            xl = ensemble_layer(x0, xl, P, l, cfg.n_heads, cfg.n_tables)
    elif cfg.backbone == "masknet":
        xl = masknet_forward(cfg, P, x0)
    else:
        raise ValueError(cfg.backbone)
    h = xl
    for i in range(len(cfg.mlp_dims)):
        h = mlp_relu(h, P[f"mlp/{i}/W"], P[f"mlp/{i}/b"])
    z = head_logit(h, P["head/w"], P["head/b"])
    return {"xL": xl, "h": h, "logit": z, "scores": sigmoid(z)}


def frontend_rows(cfg, fb, spec):
    """O11 on a raw FeatureBatch (cvr_synth.FeatureBatch): per table, text -> n-gram keys, histories ->
    the most recent max_len keys, every key -> hash_index(key, rows - 1); returns (row ids int64 [nnz],
    table-major offsets [T*B + 1], per-table pooling modes)."""
    rows, lens, modes = [], [], []
    for t, (kind, tab) in enumerate(zip(spec["kinds"], fb.tables)):
        vocab = int(cfg.rows[t]) - 1
        for b in range(fb.batch):
            if tab[0] == "text":
                keys = ngram_keys(tab[1][b], spec["ngram"])
            else:
                keys = [int(x) for x in tab[1][tab[2][b]:tab[2][b + 1]]]
                if kind == "seq":
                    keys = truncate_recent(keys, spec["max_len"])
            rows.extend(hash_index(k, vocab) for k in keys)
            lens.append(len(keys))
        modes.append("sum" if kind == "cat" else "mean")
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    return np.array(rows, np.int64), off, modes


def score_forward(cfg, tables: Sequence, weights: Dict, batch, validate: bool = True,
                  modes: Sequence[str] = None) -> Dict[str, np.ndarray]:
    """S2-S7 of SURVEY.md §8(a) for one batch (``cvr_synth.Batch``): pool -> normalize ->
    concat -> backbone -> MLP -> sigmoid.  Returns scores, x0, xL (fp64)."""
    P = {k: to_f64(v) for k, v in weights.items()}
    B, T = batch.batch, cfg.n_tables
    if validate:
        validate_csr(batch.indices, batch.offsets, cfg.rows, T, B)
    if modes is None:
        pooled = embedding_bag_sum(tables, batch.indices, batch.offsets, T, B, cfg.dim)
    else:
        pooled = embedding_bag(tables, batch.indices, batch.offsets, T, B, cfg.dim, modes)
    if cfg.n_dense:
        z = normalize_dense(batch.dense, P["norm/mean"], P["norm/std"])
    else:
        z = np.zeros((B, 0))
    x0 = concat_x0(pooled, z)
    out = dense_forward(cfg, P, x0)
    out["x0"] = x0
    return out
