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
    # P12: the indices / offsets the executor's kernels consumed (read back through the call block of the last
    # batch's slot) are byte-identical to the generator's -- SHA-256 over the device copies
    import hashlib
    from paper_2605_29232_b200._cvr import EXECUTOR_SLOTS as NS
    rec, bt = m.call_info((2 * len(batches) - 1) % NS), batches[-1]  # call k uses slot k % NS (device-fed calls first)
    assert rec["batch"] == bt.batch and rec["nnz"] == bt.nnz
    nbytes = {"d_indices": bt.indices.nbytes, "d_offsets": bt.offsets.nbytes, "d_dense": bt.dense.nbytes}
    for key, ref_arr in (("d_indices", bt.indices), ("d_offsets", bt.offsets), ("d_dense", bt.dense)):
        off = rec[key] - m.workspace.data_ptr()   # host-fed: the staging slots live in the ctx's workspace
        assert 0 <= off and off + nbytes[key] <= m.workspace.numel()
        dev = m.workspace[off:off + nbytes[key]]
        assert hashlib.sha256(dev.cpu().numpy().tobytes()).hexdigest() == hashlib.sha256(ref_arr.tobytes()).hexdigest()
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


def _small(name):
    if name == "c1":
        return cs.C1
    if name == "c4":
        return cs.C4.with_(rows=(20000,) * 64)
    return cs.C6.with_(rows=(4096,) * 26)


@pytest.mark.parametrize("name", ["c1", "c4", "c6"])
def test_executor_graphs_every_backbone(name):
    """The executor's graphs (one captured graph per stage, slot and grid-size bucket, the batch read from the
    per-call block) on every backbone: batches of changing size through the same graphs are bit-identical to embed +
    dense, graphs are captured once per (stage, slot, bucket), and the call block holds exactly the pointers / sizes
    of the last batch (P12: what the kernels consumed)."""
    cfg = _small(name)
    Bmax = 256 if name == "c1" else 384
    m, tabs, w = make_model(cfg, max_batch=Bmax, max_nnz=1 << 20)
    sizes = [Bmax, 7, Bmax - 1, 1, 130, Bmax]
    batches = [cs.make_batch(cfg, 300 + i, batch=B) for i, B in enumerate(sizes)]
    dev_in = [to_dev(bt) for bt in batches]
    refs = [m.dense(m.embed(i, o, bt.batch, d), bt.batch).clone() for (i, o, d), bt in zip(dev_in, batches)]
    outs = [torch.empty(bt.batch, device="cuda") for bt in batches]
    s_e, s_d = torch.cuda.Stream(), torch.cuda.Stream(priority=-1)
    torch.cuda.synchronize()
    for (i, o, d), bt, out in zip(dev_in, batches, outs):
        m.score(i, o, bt.batch, d, out, s_embed=s_e, s_dense=s_d)
    s_d.synchronize()
    assert m.status(s_d) == 0
    for k, (out, r) in enumerate(zip(outs, refs)):
        assert torch.equal(out, r), (name, k, sizes[k])
    from paper_2605_29232_b200._cvr import EXECUTOR_SLOTS as NS
    last = m.call_info((len(sizes) - 1) % NS)
    i, o, d = dev_in[-1]
    assert (last["d_indices"], last["d_offsets"], last["nnz"], last["batch"]) == \
        (i.data_ptr(), o.data_ptr(), i.numel(), sizes[-1])
    assert last["d_scores"] == outs[-1].data_ptr()
    def bucket(b):  # grid-size bucket: next power of two >= 128, capped at max_batch (cvr_ctx::bucket_rows)
        r = 128
        while r < b and r < Bmax:
            r *= 2
        return min(r, Bmax)
    # one graph per (stage, slot, bucket): embed + dense for every distinct (slot, bucket) seen, nothing more
    assert last["graph_captures"] == 2 * len({(k % NS, bucket(b)) for k, b in enumerate(sizes)})
    m.close()


@pytest.mark.parametrize("name,lanes", [("c1", 2), ("c2", 2), ("c2", 3), ("c6", 2)])
def test_executor_lanes(name, lanes):
    """Option "lanes": consecutive cvr_score / cvr_score_host calls dealt round-robin to `lanes` pipelines (sub-contexts
    on library streams, joined into the caller's s_dense): every batch's scores bit-identical to embed + dense on
    lane 0, the call blocks of the last calls are where executor_slot() says, each lane captures its own graphs,
    and a bad index in a batch dealt to a lane other than 0 still reaches cvr_get_status."""
    cfg = cs.C2.with_(rows=(50000,) * 26) if name == "c2" else _small(name)
    Bmax = 256 if name == "c1" else 384
    m, tabs, w = make_model(cfg, max_batch=Bmax, max_nnz=1 << 20, lanes=lanes)
    sizes = [Bmax, 7, Bmax - 1, 1, 130, Bmax, 64, 200]
    batches = [cs.make_batch(cfg, 400 + i, batch=B) for i, B in enumerate(sizes)]
    dev_in = [to_dev(bt) for bt in batches]
    refs = [m.dense(m.embed(i, o, bt.batch, d), bt.batch).clone() for (i, o, d), bt in zip(dev_in, batches)]
    outs = [torch.empty(bt.batch, device="cuda") for bt in batches]
    s_e, s_d, s_c = torch.cuda.Stream(), torch.cuda.Stream(priority=-1), torch.cuda.Stream()
    torch.cuda.synchronize()
    for (i, o, d), bt, out in zip(dev_in, batches, outs):
        m.score(i, o, bt.batch, d, out, s_embed=s_e, s_dense=s_d)
    s_d.synchronize()
    assert m.status(s_d) == 0
    for k, (out, r) in enumerate(zip(outs, refs)):
        assert torch.equal(out, r), (name, lanes, k, sizes[k])
    from paper_2605_29232_b200._cvr import EXECUTOR_SLOTS as NS
    n = len(sizes)
    for j in (n - 1, n - 2):
        rec = m.call_info(m.executor_slot(j))
        i, o, d = dev_in[j]
        assert (rec["d_indices"], rec["d_offsets"], rec["nnz"], rec["batch"], rec["d_scores"]) == \
            (i.data_ptr(), o.data_ptr(), i.numel(), sizes[j], outs[j].data_ptr())

    def bucket(b):
        r = 128
        while r < b and r < Bmax:
            r *= 2
        return min(r, Bmax)
    seen = {(k % lanes, (k // lanes) % NS, bucket(b)) for k, b in enumerate(sizes)}
    assert rec["graph_captures"] == 2 * len(seen)
    # host-fed through the lanes (pinned inputs, zero-copy scores), continuing the call count
    host_in = [tuple(torch.from_numpy(a).pin_memory() for a in (bt.indices, bt.offsets, bt.dense)) for bt in batches]
    houts = [torch.empty(bt.batch, dtype=torch.float32).pin_memory() for bt in batches]
    for (idx, off, dense), bt, o in zip(host_in, batches, houts):
        m.score_host(idx, off, bt.batch, dense, o, s_copy=s_c, s_embed=s_e, s_dense=s_d)
    s_d.synchronize()
    assert m.status(s_d) == 0
    for o, r in zip(houts, refs):
        assert torch.equal(o, r.cpu())
    # a malformed batch dealt to a lane other than 0 (call 2n + 1): that lane's sticky flag reaches cvr_get_status
    bad = cs.make_batch(cfg, 499, batch=64)
    bi = bad.indices.copy()
    bi[5] = 1 << 30
    good_in = to_dev(batches[0])
    m.score(*good_in[:2], batches[0].batch, good_in[2], outs[0], s_embed=s_e, s_dense=s_d)   # lane 0
    m.score(torch.from_numpy(bi).cuda(), torch.from_numpy(bad.offsets).cuda(), 64,
            torch.from_numpy(bad.dense).cuda(), outs[6], s_embed=s_e, s_dense=s_d)             # lane (2n+1) % L
    s_d.synchronize()
    from paper_2605_29232_b200._cvr import CVR_E_INDEX
    assert m.status(s_d) == CVR_E_INDEX
    assert m.status(s_d) == 0  # the flag is cleared once reported
    m.close()


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


@pytest.mark.parametrize("B", [16384, 12345])
def test_c2_many_tiles_per_cta_bitexact(B):
    """Large batches give every persistent GEMM CTA many tiles (the U GEMM's last-tile epilogue inputs go
    through the operand ring, the slots cycle many times): 192-wide ring tiles == 64-wide tiles bit-exact, and a
    sample vs the oracle.  Synthetic x0 (no tables needed for the dense stage)."""
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
    m.close()
    assert torch.equal(s192, s64)
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


def test_c3_rank_slice_dense_stage_vs_oracle():
    """The dense stage of one c3 rank at N = 8 (W = 12,864, B/N = 8,192 rows: many tiles per persistent CTA on every
    GEMM) against the oracle on a sample of 64 rows; synthetic x0 (the dense stage needs no tables)."""
    from paper_2605_29232_b200 import CvrModel
    cfg = cs.C3
    B = 8192
    w = cs.make_weights(cfg)
    m = CvrModel(cfg, max_batch=B, max_nnz=1 << 12)
    m.load_weights({k: v.cuda() for k, v in w.items()})
    x0 = m.new_x0(B).zero_()
    g = torch.Generator(device="cuda").manual_seed(11)
    x0[:, :cfg.width] = (torch.randn(B, cfg.width, device="cuda", generator=g) * 0.3).to(x0.dtype)
    s = m.dense(x0, B)
    assert m.status() == 0
    sel = np.random.default_rng(5).choice(B, 64, replace=False)
    xs = x0[torch.from_numpy(sel).cuda(), :cfg.width].double().cpu().numpy()
    ref = O.dense_forward(cfg, {k: O.to_f64(v) for k, v in w.items()}, xs)["scores"]
    err = np.abs(s[torch.from_numpy(sel).cuda()].double().cpu().numpy() - ref)
    m.close()
    assert err.max() <= TOL_BF16, err.max()


@pytest.mark.slow
def test_c2_full_size_two_lanes_vs_oracle():
    """BASELINE.json configs[1] at full size (26 tables of 1e5-1e6 rows x 64 bf16, B = 4096) in the launch configuration
    bench.py times: the executor with two lanes, four pipelined batches (two per lane, both x0 slots of lane 0 and one
    of lane 1), every one of each batch's 4096 scores against the fp64 oracle (gate 2e-3)."""
    cfg = cs.C2
    ring = [cs.make_batch(cfg, 910 + i) for i in range(4)]
    m, tabs, w = make_model(cfg, max_batch=cfg.batch, max_nnz=max(b.nnz for b in ring), lanes=2)
    dev_in = [to_dev(b) for b in ring]
    outs = [torch.empty(cfg.batch, device="cuda") for _ in ring]
    s_e, s_d = torch.cuda.Stream(), torch.cuda.Stream(priority=-1)
    torch.cuda.synchronize()
    for (i, o, d), bt, out in zip(dev_in, ring, outs):
        m.score(i, o, bt.batch, d, out, s_embed=s_e, s_dense=s_d)
    s_d.synchronize()
    assert m.status(s_d) == 0
    specs = cs.table_specs(cfg)
    for k, (bt, out) in enumerate(zip(ring, outs)):
        ref = O.score_forward(cfg, specs, w, bt)["scores"]
        err = np.abs(out.double().cpu().numpy() - ref)
        assert err.max() <= TOL_BF16, (k, err.max(), np.percentile(err, 99))
    m.close()


@pytest.mark.parametrize("lanes", [1, 2])
def test_executor_empty_batches_and_bags(lanes):
    """Edge cases through the executor: a batch of 0 rows between real batches (no work, no error, the neighbours'
    scores unchanged) and a batch whose every bag is empty (x0's embedding columns all 0: every score equals the
    oracle's on the all-empty batch), one and two lanes."""
    cfg = cs.C2.with_(rows=(5000,) * 26)
    Bmax = 256
    m, tabs, w = make_model(cfg, max_batch=Bmax, max_nnz=1 << 18, lanes=lanes)
    a = cs.make_batch(cfg, 500, batch=200)
    empty = cs.make_batch(cfg, 501, batch=130)
    empty_off = np.zeros_like(empty.offsets)                    # every bag [0, 0): nnz = 0
    dev_a = to_dev(a)
    ref_a = m.dense(m.embed(*dev_a[:2], a.batch, dev_a[2]), a.batch).clone()
    s_e, s_d = torch.cuda.Stream(), torch.cuda.Stream(priority=-1)
    out1, out2 = torch.empty(a.batch, device="cuda"), torch.empty(a.batch, device="cuda")
    oute = torch.empty(empty.batch, device="cuda")
    zero_idx = torch.zeros(1, dtype=torch.int32, device="cuda")
    zero_off = torch.zeros(cfg.n_tables * 1 + 1, dtype=torch.int32, device="cuda")
    dummy_scores = torch.empty(1, device="cuda")
    dense0 = torch.zeros(1, cfg.n_dense, device="cuda")
    torch.cuda.synchronize()
    m.score(*dev_a[:2], a.batch, dev_a[2], out1, s_embed=s_e, s_dense=s_d)
    m.L.cvr_score(m.h, zero_idx.data_ptr(), zero_off.data_ptr(), 0, 0, dense0.data_ptr(), dummy_scores.data_ptr(),
                  s_e.cuda_stream, s_d.cuda_stream)                              # batch of 0 rows
    m.score(zero_idx[:0], torch.from_numpy(empty_off).cuda(), empty.batch, torch.from_numpy(empty.dense).cuda(), oute,
            s_embed=s_e, s_dense=s_d)                                             # every bag empty
    m.score(*dev_a[:2], a.batch, dev_a[2], out2, s_embed=s_e, s_dense=s_d)
    s_d.synchronize()
    assert m.status(s_d) == 0
    assert torch.equal(out1, ref_a) and torch.equal(out2, ref_a)
    eb = cs.Batch(empty.batch, cfg.n_tables, np.zeros(0, np.int32), empty_off, empty.dense)
    ref_e = O.score_forward(cfg, cs.table_specs(cfg), w, eb)["scores"]
    assert np.abs(oute.double().cpu().numpy() - ref_e).max() <= TOL_BF16
    m.close()


@pytest.mark.parametrize("lanes", [2, 3])
def test_executor_lanes_stress(lanes):
    """Race check for the lanes: 60 batches of random size (1 .. max_batch), device-fed and host-fed calls
    interleaved at random, inputs and outputs in distinct buffers, one synchronisation at the end; every batch's
    scores bit-identical to embed + dense of the same batch."""
    cfg = cs.C2.with_(rows=(20000,) * 26)
    Bmax = 512
    m, tabs, w = make_model(cfg, max_batch=Bmax, max_nnz=1 << 20, lanes=lanes)
    rng = np.random.default_rng(7)
    sizes = rng.integers(1, Bmax + 1, 60)
    batches = [cs.make_batch(cfg, 600 + i, batch=int(b)) for i, b in enumerate(sizes)]
    dev_in = [to_dev(bt) for bt in batches]
    refs = [m.dense(m.embed(i, o, bt.batch, d), bt.batch).clone() for (i, o, d), bt in zip(dev_in, batches)]
    host = rng.random(len(batches)) < 0.4
    host_in = [tuple(torch.from_numpy(a).pin_memory() for a in (bt.indices, bt.offsets, bt.dense)) if h else None
               for bt, h in zip(batches, host)]
    outs = [torch.empty(bt.batch).pin_memory() if h else torch.empty(bt.batch, device="cuda")
            for bt, h in zip(batches, host)]
    s_e, s_d, s_c = torch.cuda.Stream(), torch.cuda.Stream(priority=-1), torch.cuda.Stream()
    torch.cuda.synchronize()
    for k, bt in enumerate(batches):
        if host[k]:
            idx, off, dense = host_in[k]
            m.score_host(idx, off, bt.batch, dense, outs[k], s_copy=s_c, s_embed=s_e, s_dense=s_d)
        else:
            i, o, d = dev_in[k]
            m.score(i, o, bt.batch, d, outs[k], s_embed=s_e, s_dense=s_d)
    s_d.synchronize()
    assert m.status(s_d) == 0
    for k, (out, r) in enumerate(zip(outs, refs)):
        assert torch.equal(out.cuda() if host[k] else out, r), (k, int(sizes[k]), bool(host[k]))
    m.close()
