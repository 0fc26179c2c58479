"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle on the same seeded
inputs.  Tolerances are BASELINE.json's north star: 1e-5 absolute on config-1 (fp32) scores,
2e-3 absolute on bf16-path sigmoid outputs; indices/offsets and single-hot bags bit-exact."""
import numpy as np
import pytest
import torch

import cvr_synth as cs
import oracle as O
from helpers import TOL_BF16, TOL_F32, device_tables, make_model, sub_batch, to_dev

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # collected on CPU hosts too; skipped there
    pytest.skip("needs a CUDA device", allow_module_level=True)


@pytest.fixture(scope="module", autouse=True)
def _build():
    from paper_2605_29232_b200 import build
    build.build()


# ------------------------------------------------------------------------------ config 1
@pytest.fixture(scope="module")
def c1():
    cfg = cs.C1
    m, tabs, w = make_model(cfg, max_batch=512, max_nnz=1 << 16)
    return cfg, m, tabs, w


@pytest.mark.parametrize("B", [256, 77, 1, 512])
def test_c1_scores_vs_oracle(c1, B):
    cfg, m, tabs, w = c1
    bt = cs.make_batch(cfg, 11, batch=B)
    idx, off, dense = to_dev(bt)
    x0 = m.embed(idx, off, B, dense)
    scores = m.dense(x0, B)
    assert m.status() == 0
    ref = O.score_forward(cfg, cs.table_specs(cfg), w, bt)
    np.testing.assert_allclose(x0[:, :cfg.width].double().cpu().numpy(), ref["x0"], rtol=0, atol=2e-6)
    assert torch.all(x0[:, cfg.width:] == 0)
    err = np.abs(scores.double().cpu().numpy() - ref["scores"]).max()
    assert err <= TOL_F32, err


def test_c1_single_hot_bitexact_and_empty_bags(c1):
    cfg, m, tabs, w = c1
    B, T = 64, cfg.n_tables
    rng = np.random.default_rng(3)
    L = rng.integers(0, 2, size=(T, B))          # empty and single-hot bags
    off = np.concatenate([[0], np.cumsum(L.ravel())]).astype(np.int32)
    idx = rng.integers(0, 1000, off[-1]).astype(np.int32)
    dense = rng.random((B, cfg.n_dense), dtype=np.float32)
    x0 = m.embed(torch.from_numpy(idx).cuda(), torch.from_numpy(off).cuda(), B, torch.from_numpy(dense).cuda())
    assert m.status() == 0
    x0 = x0.cpu()
    for t in range(T):
        for b in range(B):
            seg = idx[off[t * B + b]:off[t * B + b + 1]]
            got = x0[b, t * 16:(t + 1) * 16]
            want = tabs[t][int(seg[0])].cpu() if len(seg) else torch.zeros(16)
            assert torch.equal(got, want)


def test_c1_bad_index_sets_status_and_zeroes_bag(c1):
    cfg, m, tabs, w = c1
    bt = cs.make_batch(cfg, 1, batch=8)
    bad = bt.indices.copy()
    bad[0] = 1000                                # == rows: out of range
    x0 = m.embed(torch.from_numpy(bad).cuda(), torch.from_numpy(bt.offsets).cuda(), 8, torch.from_numpy(bt.dense).cuda())
    assert m.status() == 5                        # CVR_E_INDEX
    assert torch.all(x0[0, :16] == 0)
    assert m.status() == 0                        # sticky flag cleared by the read
    off = bt.offsets.copy()
    off[3] = off[4] + 1                          # non-monotone offsets
    m.embed(torch.from_numpy(bt.indices).cuda(), torch.from_numpy(off).cuda(), 8, torch.from_numpy(bt.dense).cuda())
    assert m.status() == 5


# ------------------------------------------------------------------------------ config 2
@pytest.fixture(scope="module")
def c2():
    cfg = cs.C2
    m, tabs, w = make_model(cfg, max_batch=4096, max_nnz=1 << 20)
    return cfg, m, tabs, w


@pytest.mark.parametrize("B", [300, 128, 1, 4096])
def test_c2_scores_vs_oracle(c2, B):
    """B=300: three 128-row tiles with a ragged tail; B=4096: config 2's full batch, checked on a
    sample of 384 examples (the oracle is row-independent, P9)."""
    cfg, m, tabs, w = c2
    bt = cs.make_batch(cfg, 5, batch=B)
    idx, off, dense = to_dev(bt)
    x0 = m.embed(idx, off, B, dense)
    scores = m.dense(x0, B)
    assert m.status() == 0
    sel = np.arange(B) if B <= 300 else np.random.default_rng(0).choice(B, 384, replace=False)
    ref = O.score_forward(cfg, cs.table_specs(cfg), w, sub_batch(bt, sel))
    x0s = x0[torch.from_numpy(sel).cuda()].double().cpu().numpy()
    # x0 is stored bf16: |delta| <= half an ulp of bf16 (2^-9 relative) + fp32 accumulation
    np.testing.assert_allclose(x0s, ref["x0"], rtol=2 ** -8, atol=1e-6)
    err = np.abs(scores[torch.from_numpy(sel).cuda()].double().cpu().numpy() - ref["scores"]).max()
    assert err <= TOL_BF16, err


def test_c2_single_hot_bitexact(c2):
    cfg, m, tabs, w = c2
    B, T = 200, cfg.n_tables
    rng = np.random.default_rng(9)
    off = np.arange(T * B + 1, dtype=np.int32)
    idx = np.concatenate([rng.integers(0, cfg.rows[t], B) for t in range(T)]).astype(np.int32)
    dense = np.zeros((B, cfg.n_dense), np.float32)
    x0 = m.embed(torch.from_numpy(idx).cuda(), torch.from_numpy(off).cuda(), B, torch.from_numpy(dense).cuda())
    assert m.status() == 0
    for t in (0, 7, 25):
        rows = tabs[t][torch.from_numpy(idx[t * B:(t + 1) * B].astype(np.int64)).cuda()]
        assert torch.equal(x0[:, t * 64:(t + 1) * 64], rows)


def test_c2_batch_invariance(c2):
    """P10: an item's score is bit-identical whichever batch (size, position) it lands in."""
    cfg, m, tabs, w = c2
    bt = cs.make_batch(cfg, 21, batch=1000)
    idx, off, dense = to_dev(bt)
    full = m.dense(m.embed(idx, off, 1000, dense), 1000)
    sel = np.array([999, 0, 517, 128, 127, 3])
    sb = sub_batch(bt, sel)
    i2, o2, d2 = to_dev(sb)
    part = m.dense(m.embed(i2, o2, len(sel), d2), len(sel))
    assert torch.equal(part, full[torch.from_numpy(sel).cuda()])


def test_c2_score_pipelined_and_host_fed_match(c2):
    """cvr_score (two streams, double-buffered x0) and cvr_score_host (pinned host buffers)
    give bit-identical scores to embed+dense, over several back-to-back batches."""
    cfg, m, tabs, w = c2
    s_e, s_d, s_c = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    batches = [cs.make_batch(cfg, 100 + i, batch=B) for i, B in enumerate([4096, 1000, 4096, 7, 2048])]
    refs = []
    for bt in batches:
        idx, off, dense = to_dev(bt)
        refs.append(m.dense(m.embed(idx, off, bt.batch, dense), bt.batch).clone())
    torch.cuda.synchronize()
    dev_in = [to_dev(bt) for bt in batches]
    outs = [torch.empty(bt.batch, device="cuda") for bt in batches]
    torch.cuda.synchronize()  # the side streams do not order after the current stream's copies
    for (idx, off, dense), bt, o in zip(dev_in, batches, outs):
        m.score(idx, off, bt.batch, dense, o, s_embed=s_e, s_dense=s_d)
    s_d.synchronize()
    for o, r in zip(outs, refs):
        assert torch.equal(o, r)
    host_in = [(torch.from_numpy(bt.indices).pin_memory(), torch.from_numpy(bt.offsets).pin_memory(),
                torch.from_numpy(bt.dense).pin_memory()) for bt in batches]
    houts = [torch.empty(bt.batch, dtype=torch.float32).pin_memory() for bt in batches]
    for (idx, off, dense), bt, o in zip(host_in, batches, houts):
        m.score_host(idx, off, bt.batch, dense, o, s_copy=s_c, s_embed=s_e, s_dense=s_d)
    s_d.synchronize()
    assert m.status(s_d) == 0
    for o, r in zip(houts, refs):
        assert torch.equal(o, r.cpu())
    # S8 variants: pinned h_scores take the zero-copy store (above); pageable h_scores and the option off take
    # the D2H copy on s_dense -- same scores
    pageable = [torch.empty(bt.batch, dtype=torch.float32) for bt in batches]
    for (idx, off, dense), bt, o in zip(host_in, batches, pageable):
        m.score_host(idx, off, bt.batch, dense, o, s_copy=s_c, s_embed=s_e, s_dense=s_d)
    s_d.synchronize()
    m.set_option("zero_copy_scores", 0)
    try:
        houts2 = [torch.empty(bt.batch, dtype=torch.float32).pin_memory() for bt in batches]
        for (idx, off, dense), bt, o in zip(host_in, batches, houts2):
            m.score_host(idx, off, bt.batch, dense, o, s_copy=s_c, s_embed=s_e, s_dense=s_d)
        s_d.synchronize()
    finally:
        m.set_option("zero_copy_scores", 1)
    for o, o2, r in zip(pageable, houts2, refs):
        assert torch.equal(o, r.cpu()) and torch.equal(o2, r.cpu())


def test_c2_zero_weights_closed_form():
    """P4 + P7 on the GPU: U = 0 makes every cross layer x_l + x0*b; zero MLP/head weights
    give score = sigmoid(head/b) exactly as the oracle's closed form."""
    cfg = cs.C2.with_(rows=(1000,) * 26)
    w = cs.make_weights(cfg)
    for k in w:
        if k.endswith("/U"):
            w[k] = torch.zeros_like(w[k])
    m, tabs, _ = make_model(cfg, max_batch=256, weights=w)
    bt = cs.make_batch(cfg, 2, batch=256)
    idx, off, dense = to_dev(bt)
    s = m.dense(m.embed(idx, off, 256, dense), 256)
    ref = O.score_forward(cfg, cs.table_specs(cfg), w, bt)
    assert np.abs(s.double().cpu().numpy() - ref["scores"]).max() <= TOL_BF16


def test_c2_fused_and_unfused_cross_agree(c2):
    """K5 (one clustered kernel per cross layer) and the two-GEMM path both meet the oracle; they differ
    only by fp32 summation order inside t = x_l V^T (K-split partials vs one accumulator)."""
    cfg, m, tabs, w = c2
    B = 520
    bt = cs.make_batch(cfg, 77, batch=B)
    idx, off, dense = to_dev(bt)
    x0 = m.embed(idx, off, B, dense)
    s_u = m.dense(x0, B).clone()
    m.set_option("fused_cross", 1)
    try:
        s_f = m.dense(x0, B).clone()
    finally:
        m.set_option("fused_cross", 0)
    ref = O.score_forward(cfg, cs.table_specs(cfg), w, bt)["scores"]
    for s in (s_f, s_u):
        assert np.abs(s.double().cpu().numpy() - ref).max() <= TOL_BF16
    assert (s_f - s_u).abs().max().item() <= 5e-4


def test_c2_a_resident_bitexact(c2):
    """The resident-A U GEMM (contiguous tile runs, t loaded once per m-block) computes exactly the same
    MMAs in the same K order as the streaming variant: bit-identical scores."""
    cfg, m, tabs, w = c2
    B = 777
    bt = cs.make_batch(cfg, 31, batch=B)
    idx, off, dense = to_dev(bt)
    x0 = m.embed(idx, off, B, dense)
    s_st = m.dense(x0, B).clone()
    m.set_option("a_resident", 1)
    try:
        s_ar = m.dense(x0, B).clone()
    finally:
        m.set_option("a_resident", 0)
    assert torch.equal(s_ar, s_st)


@pytest.mark.parametrize("B", [4096, 333])
def test_c2_cross_stack_bitexact(c2, B):
    """The persistent dependency-driven cross stack runs the same tiles, K order and epilogue as the
    per-GEMM launches: bit-identical scores, for a full and a ragged batch."""
    cfg, m, tabs, w = c2
    bt = cs.make_batch(cfg, 41, batch=B)
    idx, off, dense = to_dev(bt)
    x0 = m.embed(idx, off, B, dense)
    s_plain = m.dense(x0, B).clone()
    m.set_option("stack", 1)
    try:
        s_stack = m.dense(x0, B).clone()
    finally:
        m.set_option("stack", 0)
    assert torch.equal(s_stack, s_plain)


@pytest.mark.parametrize("B", [4096, 333])
def test_c2_multicast_clusters(c2, B):
    """A-multicast clusters (option "mc"): mc = 2 (every grouped GEMM multicast, same per-tile MMAs and K order)
    and mc = 1 (the head as a 4-CTA cluster summing its 64-column partial dot products over DSMEM in rank order) are
    bit-identical to the default mc = 0 (the head as one 256-wide tile whose split epilogue sums the same 64-column
    partials in the same order); all meet the oracle."""
    cfg, m, tabs, w = c2
    bt = cs.make_batch(cfg, 43, batch=B)
    idx, off, dense = to_dev(bt)
    x0 = m.embed(idx, off, B, dense)
    s1 = m.dense(x0, B).clone()
    try:
        m.set_option("mc", 2)
        s2 = m.dense(x0, B).clone()
        m.set_option("mc", 1)
        s0 = m.dense(x0, B).clone()
    finally:
        m.set_option("mc", 0)
    assert torch.equal(s2, s1)
    assert torch.equal(s0, s1)
    sel = np.arange(B) if B <= 333 else np.random.default_rng(1).choice(B, 256, replace=False)
    ref = O.score_forward(cfg, cs.table_specs(cfg), w, sub_batch(bt, sel))["scores"]
    assert np.abs(s1[torch.from_numpy(sel).cuda()].double().cpu().numpy() - ref).max() <= TOL_BF16


@pytest.mark.parametrize("B", [4096, 333])
def test_c2_u_tile_192_bitexact(c2, B):
    """U GEMM at 192-wide tiles (EIN-ring epilogue, in-place x_{l+1}) vs 64-wide tiles: each output element
    sees the same MMAs in the same K order and the same fp32 epilogue -> bit-identical scores; both meet the
    oracle."""
    cfg, m, tabs, w = c2
    bt = cs.make_batch(cfg, 47, batch=B)
    idx, off, dense = to_dev(bt)
    x0 = m.embed(idx, off, B, dense)
    s192 = m.dense(x0, B).clone()
    m.set_option("u_bn", 64)
    try:
        s64 = m.dense(x0, B).clone()
    finally:
        m.set_option("u_bn", 192)
    assert torch.equal(s192, s64)
    sel = np.arange(B) if B <= 333 else np.random.default_rng(2).choice(B, 256, replace=False)
    ref = O.score_forward(cfg, cs.table_specs(cfg), w, sub_batch(bt, sel))["scores"]
    assert np.abs(s192[torch.from_numpy(sel).cuda()].double().cpu().numpy() - ref).max() <= TOL_BF16


@pytest.mark.parametrize("B", [4096, 333, 1])
def test_c2_xv_splitk(c2, B):
    """t = x_l V^T as a K-split cluster GEMM (4 partials summed in DSMEM in a fixed order) vs one 128 x 64
    tile accumulator: both meet the oracle, and they agree to fp32 summation-order rounding of t."""
    cfg, m, tabs, w = c2
    bt = cs.make_batch(cfg, 53, batch=B)
    idx, off, dense = to_dev(bt)
    x0 = m.embed(idx, off, B, dense)
    s_tile = m.dense(x0, B).clone()
    try:
        m.set_option("xv_splitk", 1)
        s_split = m.dense(x0, B).clone()
        m.set_option("xv_splitk", 2)  # partials exchanged through L2 instead of DSMEM: same sums, same order
        s_split2 = m.dense(x0, B).clone()
    finally:
        m.set_option("xv_splitk", 0)
    assert torch.equal(s_split, s_split2)
    assert (s_split - s_tile).abs().max().item() <= 5e-4
    sel = np.arange(B) if B <= 333 else np.random.default_rng(3).choice(B, 256, replace=False)
    ref = O.score_forward(cfg, cs.table_specs(cfg), w, sub_batch(bt, sel))["scores"]
    for s in (s_split, s_tile):
        assert np.abs(s[torch.from_numpy(sel).cuda()].double().cpu().numpy() - ref).max() <= TOL_BF16


@pytest.mark.parametrize("B", [4096, 333, 1])
def test_c2_weight_multicast_bitexact(c2, B):
    """Option mb: weight tiles sliced and TMA-multicast over clusters of 8 row blocks (padded row-block count
    for ragged batches).  Only the load routing changes: bit-identical scores."""
    cfg, m, tabs, w = c2
    bt = cs.make_batch(cfg, 59, batch=B)
    idx, off, dense = to_dev(bt)
    x0 = m.embed(idx, off, B, dense)
    s0 = m.dense(x0, B).clone()
    m.set_option("mb", 1)
    try:
        s1 = m.dense(x0, B).clone()
    finally:
        m.set_option("mb", 0)
    assert torch.equal(s0, s1)


@pytest.mark.parametrize("B", [4096, 333])
def test_c2_pair_mlp_bitexact(c2, B):
    """Option pair_mlp: the hidden MLP GEMMs as 2-CTA (cta_group::2) 256-row tiles with split epilogues; same
    MMAs per output element in the same K order -> bit-identical scores."""
    cfg, m, tabs, w = c2
    bt = cs.make_batch(cfg, 61, batch=B)
    idx, off, dense = to_dev(bt)
    x0 = m.embed(idx, off, B, dense)
    s0 = m.dense(x0, B).clone()
    m.set_option("pair_mlp", 1)
    try:
        s1 = m.dense(x0, B).clone()
    finally:
        m.set_option("pair_mlp", 0)
    assert torch.equal(s0, s1)


@pytest.mark.parametrize("bn", [64, 128, 256])
@pytest.mark.parametrize("B", [4096, 333])
def test_c2_pair_xv_bitexact(c2, B, bn):
    """Option pair_xv: t = x_l V^T as 2-CTA (cta_group::2) 256 x BN tiles; same MMAs per output element in the
    same K order -> bit-identical scores."""
    cfg, m, tabs, w = c2
    bt = cs.make_batch(cfg, 62, batch=B)
    idx, off, dense = to_dev(bt)
    x0 = m.embed(idx, off, B, dense)
    s0 = m.dense(x0, B).clone()
    m.set_option("pair_xv", bn)
    try:
        s1 = m.dense(x0, B).clone()
    finally:
        m.set_option("pair_xv", 0)
    assert torch.equal(s0, s1)



@pytest.mark.parametrize("bn", [128, 256])
def test_c2_xv_bn_bitexact(c2, bn):
    """Option xv_bn (the xV N tile; the default picks it by wave count, pick_bn_xv): every tile width runs the
    same K order per output element -> bit-identical scores, ragged batch included."""
    cfg, m, tabs, w = c2
    for B in (4096, 333):
        bt = cs.make_batch(cfg, 64, batch=B)
        idx, off, dense = to_dev(bt)
        x0 = m.embed(idx, off, B, dense)
        s0 = m.dense(x0, B).clone()
        m.set_option("xv_bn", bn)
        try:
            s1 = m.dense(x0, B).clone()
        finally:
            m.set_option("xv_bn", 0)
        assert torch.equal(s0, s1)


@pytest.mark.parametrize("B", [4096, 333, 1])
def test_c2_pair_u_bitexact(c2, B):
    """Option pair_u: the U GEMM's 192-wide EIN-ring tiles as 2-CTA (cta_group::2) 256-row tiles, each CTA
    holding half of the U tile; same MMAs per output element in the same K order -> bit-identical scores."""
    cfg, m, tabs, w = c2
    bt = cs.make_batch(cfg, 65, batch=B)
    idx, off, dense = to_dev(bt)
    x0 = m.embed(idx, off, B, dense)
    s0 = m.dense(x0, B).clone()
    m.set_option("pair_u", 1)
    try:
        s1 = m.dense(x0, B).clone()
    finally:
        m.set_option("pair_u", 0)
    assert torch.equal(s0, s1)


@pytest.mark.parametrize("B", [16384, 12345])
def test_c2_many_tiles_per_cta_bitexact(B):
    """Large batches give every persistent GEMM CTA many tiles (the U GEMM's last-tile epilogue inputs go
    through the operand ring, the slots cycle many times): 192-wide ring tiles == 64-wide tiles bit-exact, and
    2-CTA U tiles bit-exact, and a sample vs the oracle.  Synthetic x0 (no tables needed for the dense stage)."""
    from paper_2605_29232_b200 import CvrModel
    cfg = cs.C2
    w = cs.make_weights(cfg)
    m = CvrModel(cfg, max_batch=B, max_nnz=1 << 12)
    m.load_weights({k: v.cuda() for k, v in w.items()})
    x0 = m.new_x0(B)
    g = torch.Generator(device="cuda").manual_seed(7)
    x0[:, :cfg.width] = (torch.randn(B, cfg.width, device="cuda", generator=g) * 0.3).to(x0.dtype)
    s192 = m.dense(x0, B).clone()
    m.set_option("u_bn", 64)
    s64 = m.dense(x0, B).clone()
    m.set_option("u_bn", 192)
    m.set_option("pair_u", 1)
    s_pair = m.dense(x0, B).clone()
    m.close()
    assert torch.equal(s192, s64)
    assert torch.equal(s192, s_pair)
    sel = np.random.default_rng(4).choice(B, 48, replace=False)
    xs = x0[torch.from_numpy(sel).cuda(), :cfg.width].double().cpu().numpy()
    ref = O.dense_forward(cfg, {k: O.to_f64(v) for k, v in w.items()}, xs)["scores"]
    assert np.abs(s192[torch.from_numpy(sel).cuda()].double().cpu().numpy() - ref).max() <= TOL_BF16


def test_c2_api_error_paths(c2):
    """The boundary's error convention (cvr.h): host-side validation returns a status and never
    launches -- batch > max_batch and unknown options -> CVR_E_ARG, a weight of the wrong shape / an unknown name ->
    CVR_E_SHAPE -- and batch 0 is a no-op; the context stays usable afterwards (scores unchanged)."""
    from paper_2605_29232_b200._cvr import CvrError
    cfg, m, tabs, w = c2
    bt = cs.make_batch(cfg, 70, batch=64)
    idx, off, dense = to_dev(bt)
    x0 = m.embed(idx, off, 64, dense)
    s_before = m.dense(x0, 64).clone()
    big = torch.zeros(4097, 1792, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(CvrError) as e:
        m.dense(big, 4097)
    assert e.value.status == 1                                   # CVR_E_ARG
    with pytest.raises(CvrError) as e:
        m.set_option("no_such_option", 1)
    assert e.value.status == 1
    bad = {"mlp/0/W": torch.zeros(1024, 1000, dtype=torch.bfloat16, device="cuda")}
    with pytest.raises(CvrError) as e:
        m.load_weights(bad)
    assert e.value.status == 2                                   # CVR_E_SHAPE
    with pytest.raises(CvrError) as e:
        m.load_weights({"mlp/9/W": torch.zeros(8, 8, dtype=torch.bfloat16, device="cuda")})
    assert e.value.status == 2
    sc = torch.full((4,), -1.0, device="cuda")
    m.dense(x0, 0, scores=sc)                                    # batch 0: nothing to do (pointers still checked)
    assert torch.all(sc == -1.0)
    assert m.status() == 0
    assert torch.equal(m.dense(x0, 64), s_before)
