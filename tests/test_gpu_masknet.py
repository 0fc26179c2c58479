"""GPU parity of the MaskNet backbone through the C ABI against the
fp64 oracle (oracle.masknet_forward): config c6 (c2 features, cross width 2048, 2 parallel blocks, mask
hidden 512, MLP 1024-512-256) and a sequential variant, bf16 tolerance 2e-3 (BASELINE.json's bf16 gate),
zero-mask closed form, batch invariance."""
import numpy as np
import pytest
import torch

import cvr_synth as cs
import oracle as O
from helpers import TOL_BF16, make_model, sub_batch, to_dev

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)


@pytest.fixture(scope="module", autouse=True)
def _build():
    from paper_2605_29232_b200 import build
    build.build()


@pytest.fixture(scope="module")
def c6():
    cfg = cs.C6
    m, tabs, w = make_model(cfg, max_batch=4096, max_nnz=1 << 20)
    return cfg, m, tabs, w


@pytest.mark.parametrize("B", [300, 1, 4096])
def test_c6_scores_vs_oracle(c6, B):
    cfg, m, tabs, w = c6
    bt = cs.make_batch(cfg, 7, batch=B)
    idx, off, dense = to_dev(bt)
    scores = m.dense(m.embed(idx, off, B, dense), B)
    assert m.status() == 0
    sel = np.arange(B) if B <= 300 else np.random.default_rng(0).choice(B, 256, replace=False)
    ref = O.score_forward(cfg, cs.table_specs(cfg), w, sub_batch(bt, sel))["scores"]
    err = np.abs(scores[torch.from_numpy(sel).cuda()].double().cpu().numpy() - ref).max()
    assert err <= TOL_BF16, err


def test_c6_batch_invariance(c6):
    cfg, m, tabs, w = c6
    bt = cs.make_batch(cfg, 8, batch=700)
    idx, off, dense = to_dev(bt)
    full = m.dense(m.embed(idx, off, 700, dense), 700).clone()
    sel = np.array([699, 0, 128, 127, 333])
    i2, o2, d2 = to_dev(sub_batch(bt, sel))
    part = m.dense(m.embed(i2, o2, len(sel), d2), len(sel))
    assert torch.equal(part, full[torch.from_numpy(sel).cuda()])


def test_c6_zero_mask_closed_form():
    """U = 0 and b = 0 in every block -> every branch outputs 0 (PAPER.md:226 with a zero mask) ->
    every example's score is sigmoid(head(MLP(0))), computed here in fp64 from the stored MLP weights."""
    cfg = cs.C6.with_(mlp_dims=(256,))
    w = cs.make_weights(cfg)
    for k in list(w):
        if k.startswith("mask/") and (k.endswith("/U") or k.endswith("/b")):
            w[k] = torch.zeros_like(w[k])
    m, tabs, _ = make_model(cfg, max_batch=256, max_nnz=1 << 16, weights=w)
    bt = cs.make_batch(cfg, 9, batch=200)
    idx, off, dense = to_dev(bt)
    s = m.dense(m.embed(idx, off, 200, dense), 200).double().cpu().numpy()
    P = {k: O.to_f64(v) for k, v in w.items()}
    h = O.mlp_relu(np.zeros((1, 2 * cfg.cross_width)), P["mlp/0/W"], P["mlp/0/b"])
    want = O.sigmoid(O.head_logit(h, P["head/w"], P["head/b"]))[0]
    assert np.abs(s - want).max() <= 1e-5
    m.close()


def test_masknet_sequential_and_mixed_vs_oracle():
    """Mixed mode (SPEC.md: a sequential chain inside each parallel branch): 2 branches x 2 blocks, smaller
    widths, ragged batch."""
    cfg = cs.C6.with_(name="c6seq", n_parallel=2, n_cross=2, cross_width=512, cross_rank=128, mlp_dims=(256, 128))
    m, tabs, w = make_model(cfg, max_batch=512, max_nnz=1 << 18)
    B = 333
    bt = cs.make_batch(cfg, 11, batch=B)
    idx, off, dense = to_dev(bt)
    s = m.dense(m.embed(idx, off, B, dense), B)
    ref = O.score_forward(cfg, cs.table_specs(cfg), w, bt)["scores"]
    assert np.abs(s.double().cpu().numpy() - ref).max() <= TOL_BF16
    m.close()


@pytest.mark.parametrize("B", [4096, 333])
def test_c6_grouped_mask_launch_bitexact(c6, B):
    """The parallel branches' mask GEMMs as one grouped launch (branch g = n / W' reads H columns
    [g r, (g+1) r) and U_g) vs one launch per branch: same MMAs, same K order -> bit-identical."""
    cfg, m, tabs, w = c6
    bt = cs.make_batch(cfg, 17, batch=B)
    idx, off, dense = to_dev(bt)
    x0 = m.embed(idx, off, B, dense)
    s_g = m.dense(x0, B).clone()
    m.set_option("mask_grouped", 0)
    try:
        s_b = m.dense(x0, B).clone()
    finally:
        m.set_option("mask_grouped", 1)
    assert torch.equal(s_g, s_b)
