"""Pins for the fp64 oracle against values fixed by the paper and by mathematics
(SURVEY.md §8(c) P1-P9, P13, P16), never against the oracle itself.  CPU only."""
import json
import math
import os

import numpy as np
import pytest
import torch

import cvr_synth as cs
import oracle as O
from oracle.brute import brute_score_one

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ---- P1: hand-computed goldens ------------------------------------------------------
def test_E1_embedding_bag():
    g = gold("E1_embedding_bag.json")
    tab = np.array(g["table"], float)
    p = O.embedding_bag_sum([tab], np.array(g["indices"]), np.array(g["offsets"]), 1, 4, 2)
    assert p.shape == (4, 1, 2)
    np.testing.assert_array_equal(p[:, 0, :], np.array(g["pooled"], float))


def test_E2_cross_full():
    for c in gold("E2_cross_full.json")["cases"]:
        out = O.cross_full(np.array([c["x0"]], float), np.array([c["xl"]], float), np.array(c["W"], float),
                           np.array(c["b"], float))
        np.testing.assert_array_equal(out[0], np.array(c["out"], float), err_msg=c["derivation"])


def test_E3_cross_lowrank():
    for c in gold("E3_cross_lowrank.json")["cases"]:
        out = O.cross_lowrank(np.array([c["x0"]], float), np.array([c["xl"]], float), np.array(c["U"], float),
                              np.array(c["V"], float), np.array(c["b"], float))
        np.testing.assert_array_equal(out[0], np.array(c["out"], float), err_msg=c["derivation"])


def test_E4_end_to_end():
    g = gold("E4_end_to_end.json")
    tabs = [np.array(t, float) for t in g["tables"]]
    pooled = O.embedding_bag_sum(tabs, np.array(g["indices"]), np.array(g["offsets"]), 2, 1, 2)
    z = O.normalize_dense(np.array(g["dense"]), np.array(g["norm_mean"]), np.array(g["norm_std"]))
    x0 = O.concat_x0(pooled, z)
    np.testing.assert_array_equal(x0[0], g["x0"])
    x1 = O.cross_full(x0, x0, np.array(g["cross_W"], float), np.array(g["cross_b"], float))
    np.testing.assert_array_equal(x1[0], g["x1"])
    s0 = O.sigmoid(O.head_logit(x1, np.array(g["head_w"], float), np.array([-2.75])))
    assert s0[0] == 0.5
    s1 = O.sigmoid(O.head_logit(x1, np.array(g["head_w"], float), np.array([math.log(3) - 2.75])))
    assert abs(s1[0] - 0.75) < 1e-15


def test_E5_relu_layer():
    g = gold("E5_relu_layer.json")
    out = O.mlp_relu(np.array([g["h"]], float), np.array(g["M"], float), np.array(g["c"], float))
    np.testing.assert_array_equal(out[0], g["out"])


def test_N1_normalize():
    g = gold("N1_normalize.json")
    assert O.normalize_dense(np.array([[g["x"]]]), np.array([g["mean"]]), np.array([g["std"]]))[0, 0] == g["z"]


# ---- sigmoid closed forms (A16) ----------------------------------------------------
def test_sigmoid_closed_forms():
    z = np.array([0.0, math.log(3.0), -math.log(3.0), 40.0, -800.0, 800.0])
    s = O.sigmoid(z)
    assert s[0] == 0.5
    assert abs(s[1] - 0.75) < 1e-15 and abs(s[2] - 0.25) < 1e-15
    assert s[4] == 0.0 and s[5] == 1.0 and np.all(np.isfinite(s))
    zz = np.linspace(-30, 30, 1001)
    np.testing.assert_allclose(O.sigmoid(zz) + O.sigmoid(-zz), 1.0, rtol=0, atol=1e-15)
    # against the textbook logistic via tanh: sigma(z) = (1 + tanh(z/2)) / 2
    np.testing.assert_allclose(O.sigmoid(zz), 0.5 * (1 + np.tanh(zz / 2)), rtol=1e-14, atol=1e-16)


# ---- P2 / P3: pooling invariants -----------------------------------------------------
def test_P2_single_hot_equals_row():
    spec = cs.TableSpec(123, 3, 5000, 64, "bf16")
    ids = np.array([0, 17, 4999, 17])
    p = O.embedding_bag_sum([spec], ids, np.arange(5), 1, 4, 64)
    rows = spec.gather(ids).to(torch.float64).numpy()
    np.testing.assert_array_equal(p[:, 0, :], rows)


def test_P3_pool_order_independent_bitexact():
    rng = np.random.default_rng(0)
    for dt in ("f32", "bf16", "f16"):
        spec = cs.TableSpec(7, 1, 20000, 64, dt)
        tab = spec.materialize().to(torch.float64).numpy()
        B = 200
        L = rng.integers(0, 300, B)
        off = np.concatenate([[0], np.cumsum(L)])
        idx = rng.integers(0, 20000, off[-1])
        p1 = O.embedding_bag_sum([tab], idx, off, 1, B, 64)
        # permute within every bag (two different orders)
        for _ in range(2):
            idx2 = idx.copy()
            for b in range(B):
                seg = idx2[off[b]:off[b + 1]]
                rng.shuffle(seg)
            p2 = O.embedding_bag_sum([tab], idx2, off, 1, B, 64)
            if dt == "f32":  # fp32 rows can hold tiny values: equal up to fp64 reordering only
                np.testing.assert_allclose(p1, p2, rtol=1e-15, atol=1e-300)
            else:
                np.testing.assert_array_equal(p1, p2)


# ---- P4 / P5 / P6: cross-layer algebra -------------------------------------------------
def test_P4_zero_cross_weight():
    rng = np.random.default_rng(1)
    x0, xl, b = rng.normal(size=(5, 7)), rng.normal(size=(5, 7)), rng.normal(size=7)
    np.testing.assert_array_equal(O.cross_full(x0, xl, np.zeros((7, 7)), b), x0 * b + xl)
    np.testing.assert_array_equal(O.cross_lowrank(x0, xl, np.zeros((7, 3)), rng.normal(size=(3, 7)), b), x0 * b + xl)
    np.testing.assert_allclose(O.cross_full(x0, x0, np.zeros((7, 7)), b), x0 * (1 + b), rtol=1e-15, atol=1e-15)
    np.testing.assert_array_equal(O.cross_full(x0, xl, np.zeros((7, 7)), np.zeros(7)), xl)


def test_P5_identity_cross():
    rng = np.random.default_rng(2)
    x0 = rng.normal(size=(4, 6))
    np.testing.assert_array_equal(O.cross_full(x0, x0, np.eye(6), np.zeros(6)), x0 * x0 + x0)


def test_P6_lowrank_equals_fullrank():
    rng = np.random.default_rng(3)
    U, V = rng.normal(size=(9, 4)), rng.normal(size=(4, 9))
    x0, xl, b = rng.normal(size=(6, 9)), rng.normal(size=(6, 9)), rng.normal(size=9)
    np.testing.assert_allclose(O.cross_lowrank(x0, xl, U, V, b), O.cross_full(x0, xl, U @ V, b), rtol=1e-12, atol=1e-12)


# ---- P7: zero MLP / head weights -----------------------------------------------------
def test_P7_zero_mlp_head():
    cfg = cs.C1
    W = {k: O.to_f64(v) for k, v in cs.make_weights(cfg).items()}
    for k in list(W):
        if k.startswith("mlp/") or k == "head/w":
            W[k] = np.zeros_like(W[k])
    x0 = np.random.default_rng(4).normal(size=(8, cfg.width))
    out = O.dense_forward(cfg, W, x0)
    np.testing.assert_array_equal(out["h"], np.tile(np.maximum(W["mlp/1/b"], 0), (8, 1)))
    c = W["head/b"][0]
    np.testing.assert_array_equal(out["scores"], 1 / (1 + math.exp(-c)) if c >= 0 else math.exp(c) / (1 + math.exp(c)))


# ---- P8: batched oracle vs scalar brute force ------------------------------------------
@pytest.mark.parametrize("cfgname,B,examples", [("c1", 256, [0, 1, 100, 255]), ("c2small", 64, [0, 63])])
def test_P8_batched_vs_brute(cfgname, B, examples):
    if cfgname == "c1":
        cfg = cs.C1
    else:  # config-2 structure at a width the scalar loops finish quickly
        cfg = cs.C2.with_(name="c2small", n_tables=4, rows=cs.C2.rows[:4], n_dense=8, cross_rank=16,
                          mlp_dims=(32, 16, 8), batch=B)
    tabs = cs.table_specs(cfg)
    w = cs.make_weights(cfg)
    bt = cs.make_batch(cfg, 0, batch=B)
    out = O.score_forward(cfg, tabs, w, bt)
    P = {k: O.to_f64(v) for k, v in w.items()}
    for b in examples:
        s = brute_score_one(cfg, tabs, P, bt.indices, bt.offsets, bt.dense[b], b, B)
        assert abs(s - out["scores"][b]) <= 1e-12 * max(1.0, abs(s))


# ---- P9: batch independence (row-wise semantics) ---------------------------------------
def test_P9_batch_independence():
    cfg = cs.C1
    tabs = [t.materialize().to(torch.float64).numpy() for t in cs.table_specs(cfg)]
    w = cs.make_weights(cfg)
    bt = cs.make_batch(cfg, 0)
    full = O.score_forward(cfg, tabs, w, bt)["scores"]
    # the same examples scored as a sub-batch give bit-identical scores
    sel = np.array([5, 77, 200])
    T, B = cfg.n_tables, bt.batch
    idx, off = [], [0]
    for t in range(T):
        for b in sel:
            seg = bt.indices[bt.offsets[t * B + b]:bt.offsets[t * B + b + 1]]
            idx.extend(seg)
            off.append(off[-1] + len(seg))
    sub = cs.Batch(len(sel), T, np.array(idx, np.int32), np.array(off, np.int32), bt.dense[sel])
    part = O.score_forward(cfg, tabs, w, sub)["scores"]
    # BLAS may block a 3-row and a 256-row product differently: equal up to fp64 reordering
    np.testing.assert_allclose(part, full[sel], rtol=1e-13, atol=0)


# ---- O1: validation raises (A23) -----------------------------------------------------
def test_validation_raises():
    with pytest.raises(O.OracleInputError):
        O.validate_csr(np.array([0, 5]), np.array([0, 1, 2]), [5], 1, 2)
    with pytest.raises(O.OracleInputError):
        O.validate_csr(np.array([0, 1]), np.array([0, 2, 1]), [5], 1, 2)
    with pytest.raises(O.OracleInputError):
        O.validate_csr(np.array([0, 1]), np.array([0, 1, 3]), [5], 1, 2)
    O.validate_csr(np.array([0, 4]), np.array([0, 0, 2]), [5], 1, 2)


# ---- P13: normalisation constants by quadrature ----------------------------------------
def test_norm_constants_quadrature():
    from scipy import integrate
    phi = lambda z: math.exp(-z * z / 2) / math.sqrt(2 * math.pi)
    m1 = 2 * integrate.quad(lambda z: math.log1p(10 * z) * phi(z), 0, np.inf, epsabs=1e-14, epsrel=1e-13)[0]
    m2 = 2 * integrate.quad(lambda z: math.log1p(10 * z) ** 2 * phi(z), 0, np.inf, epsabs=1e-14, epsrel=1e-13)[0]
    assert abs(m1 - cs.NORM_MEAN) < 1e-10
    assert abs(math.sqrt(m2 - m1 * m1) - cs.NORM_STD) < 1e-10
    # and the empirical moments of the generator's dense features agree within 4 s.e.
    bt = cs.make_batch(cs.C2, 0)
    x = bt.dense.astype(np.float64).ravel()
    assert abs(x.mean() - cs.NORM_MEAN) < 4 * cs.NORM_STD / math.sqrt(x.size)


# ---- P16: zero-weight ensemble layer reduces to LN(X) ----------------------------------
def test_P16_zero_ensemble_layer():
    cfg = cs.C4.with_(n_tables=4, dim=8, rows=(50,) * 4, cross_rank=4, ffn_dim=16, n_heads=2, batch=3)
    P = {k: np.zeros(tuple(s)) for k, s in cs.weight_shapes(cfg)}
    P["ens/0/ln/gamma"] = np.ones(8)
    X = np.random.default_rng(5).normal(size=(3, 32))
    Y = O.ensemble_layer(X, X, P, 0, cfg.n_heads, cfg.n_tables)
    Xt = X.reshape(3, 4, 8)
    ref = (Xt - Xt.mean(-1, keepdims=True)) / np.sqrt(Xt.var(-1, keepdims=True) + 1e-5)
    np.testing.assert_allclose(Y.reshape(3, 4, 8), ref, rtol=1e-13, atol=1e-13)


def test_mha_uniform_attention_is_mean():
    # Q = K = 0 => softmax uniform => each token's attention output = mean of V over tokens
    rng = np.random.default_rng(6)
    X = rng.normal(size=(2, 5, 8))
    Wqkv = np.zeros((24, 8))
    Wqkv[16:] = rng.normal(size=(8, 8))
    o = O.mha_tokens(X, Wqkv, np.zeros(24), np.eye(8), np.zeros(8), 2)
    v = X @ Wqkv[16:].T
    np.testing.assert_allclose(o, np.broadcast_to(v.mean(axis=1, keepdims=True), o.shape), rtol=1e-13, atol=1e-14)


# ---- MaskNet: E6 goldens, SPEC.md:259-270 closed forms, brute force -------
def test_E6_masknet_projection_and_block():
    g = gold("E6_masknet.json")
    pj = g["projection"]
    out = O.masknet_project(np.array([pj["x0"]], float), np.array(pj["W"], float), np.array(pj["b"], float))
    np.testing.assert_array_equal(out[0], pj["out"])
    bk = g["block"]
    args = [np.array(bk[k], float) for k in ("U", "V", "c", "b")]
    x0p = np.array([bk["x0p"]], float)
    out = O.masknet_block(np.array([bk["x_in"]], float), x0p, *args)
    np.testing.assert_array_equal(out[0], bk["out"], err_msg=bk["derivation"])
    out2 = O.masknet_block(out, x0p, *args)
    np.testing.assert_array_equal(out2[0], g["sequential2"]["out"], err_msg=g["sequential2"]["derivation"])


def _tiny_masknet_cfg(P=2, S=1, width=0):
    return cs.C2.with_(name="c6tiny", n_tables=1, rows=(4,), dim=2, n_dense=0, backbone="masknet", n_cross=S,
                       cross_rank=2, cross_width=width, n_parallel=P, mlp_dims=())


def test_E6_masknet_forward_parallel_and_sequential():
    g = gold("E6_masknet.json")
    bk = g["block"]
    Pm = {f"mask/{p}/{q}/{k}": np.array(bk[k], float) for p in range(2) for q in range(2) for k in ("U", "V", "c", "b")}
    x0 = np.array([bk["x0p"]], float)
    par = O.masknet_forward(_tiny_masknet_cfg(P=2, S=1), Pm, x0)
    np.testing.assert_array_equal(par[0], g["parallel2"]["out"])
    seq = O.masknet_forward(_tiny_masknet_cfg(P=1, S=2), Pm, x0)
    np.testing.assert_array_equal(seq[0], g["sequential2"]["out"])


def test_masknet_closed_forms():
    """ReLU kills the mask -> output = b * x_in (0 when b = 0); unit mask (U = 0, b = 1) ->
    x_out = x_in; 1 parallel block == 1 sequential block; 2 identical parallel blocks -> duplicated output."""
    rng = np.random.default_rng(5)
    B, W, r = 7, 12, 5
    x0p = np.abs(rng.normal(size=(B, W)))
    x_in = rng.normal(size=(B, W))
    V = -np.abs(rng.normal(size=(r, W)))      # V x0p < 0 for a non-negative x0p
    U = rng.normal(size=(W, r))
    np.testing.assert_array_equal(O.masknet_block(x_in, x0p, U, V, np.zeros(r), np.zeros(W)), np.zeros((B, W)))
    b = rng.normal(size=W)
    np.testing.assert_array_equal(O.masknet_block(x_in, x0p, U, V, np.zeros(r), b), b * x_in)
    np.testing.assert_array_equal(
        O.masknet_block(x_in, x0p, np.zeros((W, r)), rng.normal(size=(r, W)), rng.normal(size=r), np.ones(W)), x_in)
    P = {f"mask/0/0/{k}": v for k, v in zip("UVcb", (U, rng.normal(size=(r, W)), rng.normal(size=r), b))}
    for k in "UVcb":
        P[f"mask/1/0/{k}"] = P[f"mask/0/0/{k}"]
    cfgP1 = _tiny_masknet_cfg(P=1, S=1).with_(dim=W, n_tables=1)
    one = O.masknet_forward(cfgP1, P, x0p)
    np.testing.assert_array_equal(one, O.masknet_forward(cfgP1.with_(n_parallel=1, n_cross=1), P, x0p))
    two = O.masknet_forward(cfgP1.with_(n_parallel=2), P, x0p)
    np.testing.assert_array_equal(two, np.concatenate([one, one], axis=1))


def test_P8_masknet_batched_vs_brute():
    cfg = cs.C6.with_(name="c6small", n_tables=4, rows=cs.C2.rows[:4], n_dense=8, cross_rank=16, cross_width=48,
                      n_parallel=2, n_cross=2, mlp_dims=(32, 16, 8), batch=32)
    tabs = cs.table_specs(cfg)
    w = cs.make_weights(cfg)
    bt = cs.make_batch(cfg, 0, batch=32)
    out = O.score_forward(cfg, tabs, w, bt)
    P = {k: O.to_f64(v) for k, v in w.items()}
    for b in (0, 17, 31):
        s = brute_score_one(cfg, tabs, P, bt.indices, bt.offsets, bt.dense[b], b, 32)
        assert abs(s - out["scores"][b]) <= 1e-12 * max(1.0, abs(s))


# ---- feature front end: FNV-1a reference vectors, SPEC closed forms ------------
def test_E7_fnv1a_reference_vectors_and_hash_index():
    g = gold("E7_frontend.json")
    for v in g["fnv1a64"]:
        assert O.fnv1a64(v["bytes"].encode()) == int(v["hash"], 16)
    # vocab 1 -> 0, determinism; key 0 by the closed form of 8 zero bytes
    for key in (0, 1, 12345678901234567, (1 << 63) + 5):
        assert O.hash_index(key, 1) == 0
        assert O.hash_index(key, 1000) == O.hash_index(key, 1000)
    closed = (0xCBF29CE484222325 * pow(0x100000001B3, 8, 1 << 64)) % (1 << 64)
    assert O.hash_index(0, 97) == closed % 97
    # the key's bytes are big-endian: key 0x61 hashes like the byte string 00..00 61
    assert O.hash_index(0x61, 1 << 62) == O.fnv1a64(bytes(7) + b"a") % (1 << 62)
    assert O.hash_index(O.KEY_MISSING, 777) == 777  # the unseen row


def test_E7_ngrams_mean_pool_truncate():
    g = gold("E7_frontend.json")
    for c in g["ngrams"]:
        assert O.ngram_keys(c["text"].encode(), c["n"]) == c["keys"]
    mp = g["mean_pool"]
    tab = np.array(mp["table"], float)
    idx = np.concatenate([np.array(b, np.int64) for b in mp["bags"]])
    off = np.concatenate([[0], np.cumsum([len(b) for b in mp["bags"]])])
    p = O.embedding_bag([tab], idx, off, 1, len(mp["bags"]), 2, ["mean"])
    np.testing.assert_allclose(p[:, 0, :], np.array(mp["out"]), rtol=0, atol=1e-15)
    ps = O.embedding_bag([tab], idx, off, 1, len(mp["bags"]), 2, ["sum"])
    np.testing.assert_array_equal(ps[:, 0, :], O.embedding_bag_sum([tab], idx, off, 1, len(mp["bags"]), 2)[:, 0, :])
    assert O.truncate_recent(g["truncate"]["keys"], g["truncate"]["max_len"]) == g["truncate"]["out"]
    assert O.truncate_recent([7], 3) == [7]


# ---- E8: hand-derived attention / FFN / ensemble-layer goldens (A20; VERDICT r1 "c4 under-pinned") -------
def _shift_matrix(n):
    W = np.zeros((n, n))
    for i in range(n):
        W[i, (i + 1) % n] = 1.0
    return W


def test_E8_attention_two_heads():
    c = gold("E8_attention.json")["cases"][0]
    D, H = c["D"], c["n_heads"]
    X = np.array(c["X"], float)[None]                      # [1, S=2, D]
    l3 = math.log(3.0)
    Wqkv = np.concatenate([np.zeros((D, D)), np.eye(D), np.eye(D)])
    bqkv = np.concatenate([[2 * l3, 0, 0, 0, 2 * l3, 0, 0, 0], np.zeros(D), np.zeros(D)])
    out = O.mha_tokens(X, Wqkv, bqkv, _shift_matrix(D), np.array(c["bo"], float), H)
    np.testing.assert_allclose(out[0], np.array(c["out"], float), rtol=0, atol=1e-14, err_msg=c["derivation"])


def test_E8_attention_token_queries_softmax_axis():
    a, b = math.sqrt(2 * math.log(3.0)), math.sqrt(2 * math.log(7.0))
    X = np.array([[[a, 0, 0, 0], [0, b, 0, 0]]])
    Wqkv = np.concatenate([np.eye(4)] * 3)
    out = O.mha_tokens(X, Wqkv, np.zeros(12), np.eye(4), np.zeros(4), 1)
    ref = np.array([[3 * a / 4, b / 4, 0, 0], [a / 8, 7 * b / 8, 0, 0]])  # E8_attention.json cases[1]
    np.testing.assert_allclose(out[0], ref, rtol=0, atol=1e-14)


def test_E8_ffn():
    g = gold("E8_ffn_ensemble.json")["ffn"]
    out = O.ffn_tokens(np.array([[g["x"]]], float), np.array(g["W1"], float), np.array(g["b1"], float),
                       np.array(g["W2"], float), np.array(g["b2"], float))
    np.testing.assert_array_equal(out[0, 0], np.array(g["out"], float), err_msg=g["derivation"])


def test_E8_ensemble_layer_x0_differs_from_xl():
    g = gold("E8_ffn_ensemble.json")["ensemble"]
    S, D = g["tokens"], g["D"]
    P = {"ens/0/dcn/V": np.array(g["dcn_V"], float), "ens/0/dcn/U": np.array(g["dcn_U"], float),
         "ens/0/dcn/b": np.array(g["dcn_b"], float),
         "ens/0/mha/Wqkv": np.zeros((3 * D, D)), "ens/0/mha/bqkv": np.zeros(3 * D),
         "ens/0/mha/Wo": np.zeros((D, D)), "ens/0/mha/bo": np.array([1.0, -1.0]),
         "ens/0/ffn/W1": np.zeros((4, D)), "ens/0/ffn/b1": np.zeros(4), "ens/0/ffn/W2": np.zeros((D, 4)),
         "ens/0/ffn/b2": np.zeros(D), "ens/0/ln/gamma": np.array(g["gamma"], float),
         "ens/0/ln/beta": np.array(g["beta"], float)}
    Y = O.ensemble_layer(np.array([g["X0"]], float), np.array([g["Xl"]], float), P, 0, g["n_heads"], S)
    r0, r1 = 0.75 / math.sqrt(0.5625 + 1e-5), 3 / math.sqrt(9 + 1e-5)
    np.testing.assert_allclose(Y[0], [r0, 0.5 - 2 * r0, r1, 0.5 - 2 * r1], rtol=0, atol=1e-15)
    np.testing.assert_allclose(Y[0], g["out"], rtol=0, atol=1e-15, err_msg=g["derivation"])


def test_P8_ensemble_batched_vs_brute():
    """P8 on a tiny config-4 structure (2 ensemble layers, 2 heads, 4 tokens): the batched oracle against the
    scalar loops of oracle/brute.py (independent evaluation order)."""
    cfg = cs.C4.with_(name="c4tiny", n_tables=4, rows=(64,) * 4, dim=8, cross_rank=4, ffn_dim=16, n_heads=2,
                      n_cross=2, mlp_dims=(16, 8), batch=6)
    tabs = cs.table_specs(cfg)
    w = cs.make_weights(cfg)
    bt = cs.make_batch(cfg, 0, batch=6)
    out = O.score_forward(cfg, tabs, w, bt)
    P = {k: O.to_f64(v) for k, v in w.items()}
    for b in range(6):
        s = brute_score_one(cfg, tabs, P, bt.indices, bt.offsets, bt.dense[b] if bt.dense.size else [], b, 6)
        assert abs(s - out["scores"][b]) <= 1e-12 * max(1.0, abs(s))
