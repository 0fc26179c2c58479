"""Feature front end: the host batch-assembly helpers of libcvr (text n-grams,
history truncation) against the oracle's definitions (CPU), and on the GPU the fused hashed gather
(FNV-1a 64 mod vocab, unseen row, mean pooling) against oracle.frontend_rows + the fp64 oracle."""
import numpy as np
import pytest
import torch

import cvr_synth as cs
import oracle as O
from helpers import TOL_BF16, make_model

SPEC = cs.FRONTEND_C7


@pytest.fixture(scope="module")
def fb():
    from paper_2605_29232_b200 import build
    build.build()
    return cs.make_feature_batch(cs.C7, 3, batch=96)


def test_text_ngram_keys_match_oracle(fb):
    from paper_2605_29232_b200 import text_ngram_keys
    texts = fb.tables[20][1] + [b"", b"a", b"ab", b"abc", bytes(range(200, 212))]
    for n in (1, 2, 3, 8):
        keys, off = text_ngram_keys(texts, n)
        for i, t in enumerate(texts):
            assert [int(k) for k in keys[off[i]:off[i + 1]]] == O.ngram_keys(t, n)


def test_truncate_bags_match_oracle(fb):
    from paper_2605_29232_b200 import truncate_bags
    _, keys, off = fb.tables[23]
    for max_len in (0, 1, 50, 10_000):
        k2, o2 = truncate_bags(keys, off, max_len)
        for b in range(fb.batch):
            want = O.truncate_recent([int(x) for x in keys[off[b]:off[b + 1]]], max_len)
            assert [int(x) for x in k2[o2[b]:o2[b + 1]]] == want


def test_assembled_layout_matches_oracle(fb):
    from paper_2605_29232_b200 import frontend as F
    keys, off = F.assemble_keys(fb, SPEC)
    rows, off_o, modes = O.frontend_rows(cs.C7, fb, SPEC)
    np.testing.assert_array_equal(off, off_o)
    assert len(keys) == len(rows) == off[-1]
    assert modes[:20] == ["sum"] * 20 and modes[20:] == ["mean"] * 6


# ------------------------------------------------------------------------------------------ GPU
gpu = pytest.mark.gpu


def _gpu_model(cfg, B):
    from paper_2605_29232_b200 import frontend as F
    m, tabs, w = make_model(cfg, max_batch=B, max_nnz=1 << 20)
    vocab, mode = F.feature_spec(cfg, SPEC)
    m.set_feature_spec(vocab, mode)
    return m, tabs, w


@gpu
@pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")
@pytest.mark.parametrize("B", [96, 1000])
def test_c7_hashed_gather_and_scores_vs_oracle(B):
    from paper_2605_29232_b200 import frontend as F
    cfg = cs.C7
    fbb = cs.make_feature_batch(cfg, 5, batch=B)
    m, tabs, w = _gpu_model(cfg, B)
    keys, off = F.assemble_keys(fbb, SPEC)
    kd, od = torch.from_numpy(keys).cuda(), torch.from_numpy(off).cuda()
    dense = torch.from_numpy(fbb.dense).cuda()
    x0 = m.embed_keys(kd, od, B, dense)
    scores = m.dense(x0, B)
    assert m.status() == 0
    rows, off_o, modes = O.frontend_rows(cfg, fbb, SPEC)
    bt = cs.Batch(B, cfg.n_tables, rows.astype(np.int32), off_o.astype(np.int32), fbb.dense)
    sel = np.arange(B) if B <= 96 else np.random.default_rng(0).choice(B, 128, replace=False)
    ref = O.score_forward(cfg, cs.table_specs(cfg), w, cs.sub_batch(bt, sel), modes=modes)
    x0s = x0[torch.from_numpy(sel).cuda()].double().cpu().numpy()[:, :cfg.width]
    np.testing.assert_allclose(x0s, ref["x0"], rtol=2 ** -8, atol=1e-6)
    err = np.abs(scores[torch.from_numpy(sel).cuda()].double().cpu().numpy() - ref["scores"]).max()
    assert err <= TOL_BF16, err
    m.close()


@gpu
@pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")
def test_single_key_bags_bitexact_hash_and_unseen():
    """Every bag holds exactly one key: the pooled slice is bit-identical to the table row at the oracle's
    hash_index (single-hot, P2), mean or sum; KEY_MISSING lands on the unseen row vocab = rows - 1; an empty
    bag pools to 0."""
    cfg = cs.C7
    B, T = 64, cfg.n_tables
    m, tabs, w = _gpu_model(cfg, B)
    rng = np.random.default_rng(4)
    keys = rng.integers(0, 1 << 63, size=T * B, dtype=np.int64).astype(np.uint64) * np.uint64(2) + np.uint64(1)
    keys[::7] = np.uint64(0xFFFFFFFFFFFFFFFF)
    off = np.arange(T * B + 1, dtype=np.int32)
    off[1 + 5 * B + 3:] -= 1           # bag (table 5, b = 3) empty; table 5 ends one key earlier
    keys = np.delete(keys, 5 * B + 3)
    x0 = m.embed_keys(torch.from_numpy(keys.view(np.int64)).cuda(), torch.from_numpy(off).cuda(), B,
                      torch.zeros(B, cfg.n_dense, device="cuda"))
    assert m.status() == 0
    for t in (0, 5, 21, 25):
        for b in range(B):
            lo, hi = off[t * B + b], off[t * B + b + 1]
            got = x0[b, t * cfg.dim:(t + 1) * cfg.dim]
            if hi == lo:
                assert torch.count_nonzero(got) == 0
                continue
            r = O.hash_index(int(keys[lo]), int(cfg.rows[t]) - 1)
            assert torch.equal(got, tabs[t][r]), (t, b)
    m.close()
