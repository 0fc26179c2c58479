"""Scalar-loop brute force for ONE example -- TEST INFRASTRUCTURE ONLY (see oracle/__init__).

No numpy matmul, no vectorisation: plain Python floats (IEEE fp64), one loop per index,
so it checks ``oracle.score_forward`` (P8 of SURVEY.md §8(c)) through an independent
evaluation order.  Same paper passages as the batched oracle: PAPER.md:96 (pooling),
95 (standardisation), 116-119 / 225 (DCN-v2 cross), 226-233 (MaskNet), 243-258 + reading A20 (ensemble
layer: DCN || MHA || FFN, summed, per-token LayerNorm), 229-233 (MLP), north star (sigmoid).
"""
from __future__ import annotations

import math
from typing import Dict, List, Sequence


def _mat_vec(M: List[List[float]], v: List[float]) -> List[float]:
    out = []
    for row in M:
        s = 0.0
        for a, b in zip(row, v):
            s += a * b
        out.append(s)
    return out


def brute_score_one(cfg, tables: Sequence, P: Dict, indices, offsets, dense_row, b: int, batch: int) -> float:
    """Score of example ``b`` (fp64 Python floats).  ``tables[t]`` supports ``gather_f64`` or
    indexing; ``P`` holds fp64 numpy parameters (``oracle.to_f64`` of the stored values)."""
    T, d = cfg.n_tables, cfg.dim
    x0: List[float] = []
    for t in range(T):
        lo, hi = int(offsets[t * batch + b]), int(offsets[t * batch + b + 1])
        acc = [0.0] * d
        for j in range(lo, hi):
            r = int(indices[j])
            tab = tables[t]
            row = tab.gather_f64([r])[0] if hasattr(tab, "gather_f64") else tab[r]
            for c in range(d):
                acc[c] += float(row[c])
        x0.extend(acc)
    for f in range(cfg.n_dense):
        sd = max(float(P["norm/std"][f]), 1e-8)
        x0.append((float(dense_row[f]) - float(P["norm/mean"][f])) / sd)

    tolist = lambda a: [[float(v) for v in r] for r in a] if getattr(a, "ndim", 1) == 2 else [float(v) for v in a]
    xl = list(x0)
    if cfg.backbone == "dcn_full":
        for l in range(cfg.n_cross):
            y = _mat_vec(tolist(P[f"dcn/{l}/W"]), xl)
            bb = tolist(P[f"dcn/{l}/b"])
            xl = [x0[i] * (y[i] + bb[i]) + xl[i] for i in range(len(xl))]
    elif cfg.backbone == "dcn_lowrank":
        for l in range(cfg.n_cross):
            t_ = _mat_vec(tolist(P[f"dcn/{l}/V"]), xl)
            y = _mat_vec(tolist(P[f"dcn/{l}/U"]), t_)
            bb = tolist(P[f"dcn/{l}/b"])
            xl = [x0[i] * (y[i] + bb[i]) + xl[i] for i in range(len(xl))]
    elif cfg.backbone == "masknet":  # PAPER.md:226-233, biases per A27
        if cfg.cross_width:
            y = _mat_vec(tolist(P["proj/W"]), x0)
            bb = tolist(P["proj/b"])
            x0p = [max(0.0, y[i] + bb[i]) for i in range(len(y))]
        else:
            x0p = list(x0)
        cat: List[float] = []
        for p in range(cfg.n_parallel):
            x = list(x0p)
            for q in range(cfg.n_cross):
                g = lambda n: tolist(P[f"mask/{p}/{q}/{n}"])
                hv = _mat_vec(g("V"), x0p)
                cv = g("c")
                hid = [max(0.0, hv[k] + cv[k]) for k in range(len(hv))]
                mv = _mat_vec(g("U"), hid)
                bv = g("b")
                x = [(mv[i] + bv[i]) * x[i] for i in range(len(x))]
            cat.extend(x)
        xl = cat
    elif cfg.backbone == "ensemble":  # A20: Y = LN_token(DCN + MHA + FFN), x0 = layer-0 input
        S, D, H = cfg.n_tables, d, cfg.n_heads
        dh = D // H
        for l in range(cfg.n_cross):
            g = lambda n: tolist(P[f"ens/{l}/{n}"])
            # DCN on the flattened S*D vector
            t_ = _mat_vec(g("dcn/V"), xl)
            y = _mat_vec(g("dcn/U"), t_)
            bb = g("dcn/b")
            dcn = [x0[i] * (y[i] + bb[i]) + xl[i] for i in range(len(xl))]
            toks = [xl[s * D:(s + 1) * D] for s in range(S)]
            Wqkv, bqkv = g("mha/Wqkv"), g("mha/bqkv")
            qkv = []
            for s in range(S):
                v = _mat_vec(Wqkv, toks[s])
                qkv.append([v[i] + bqkv[i] for i in range(3 * D)])
            att = [[0.0] * D for _ in range(S)]
            for h in range(H):
                for i in range(S):
                    logit = []
                    for j in range(S):
                        acc = 0.0
                        for c in range(dh):
                            acc += qkv[i][h * dh + c] * qkv[j][D + h * dh + c]
                        logit.append(acc / math.sqrt(dh))
                    mx = max(logit)
                    e = [math.exp(v - mx) for v in logit]
                    den = sum(e)
                    for c in range(dh):
                        acc = 0.0
                        for j in range(S):
                            acc += e[j] / den * qkv[j][2 * D + h * dh + c]
                        att[i][h * dh + c] = acc
            Wo, bo = g("mha/Wo"), g("mha/bo")
            W1, b1, W2, b2 = g("ffn/W1"), g("ffn/b1"), g("ffn/W2"), g("ffn/b2")
            gam, bet = g("ln/gamma"), g("ln/beta")
            out: List[float] = []
            for s in range(S):
                mo = _mat_vec(Wo, att[s])
                hid = _mat_vec(W1, toks[s])
                hid = [max(0.0, hid[k] + b1[k]) for k in range(len(hid))]
                f = _mat_vec(W2, hid)
                ysum = [dcn[s * D + c] + mo[c] + bo[c] + f[c] + b2[c] for c in range(D)]
                mu = sum(ysum) / D
                var = sum((v - mu) * (v - mu) for v in ysum) / D
                out.extend((ysum[c] - mu) / math.sqrt(var + 1e-5) * gam[c] + bet[c] for c in range(D))
            xl = out
    else:
        raise NotImplementedError("brute force covers the DCN-v2, MaskNet and ensemble configs")
    h = xl
    for i in range(len(cfg.mlp_dims)):
        y = _mat_vec(tolist(P[f"mlp/{i}/W"]), h)
        c = tolist(P[f"mlp/{i}/b"])
        h = [max(0.0, y[j] + c[j]) for j in range(len(y))]
    m = tolist(P["head/w"])[0]
    z = sum(m[j] * h[j] for j in range(len(h))) + float(P["head/b"][0])
    return 1.0 / (1.0 + math.exp(-z)) if z >= 0 else math.exp(z) / (1.0 + math.exp(z))
