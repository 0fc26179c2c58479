"""Sharded-table path on one GPU: N ranks emulated in sequence (their kernels do not wait on each
other), the all-to-all emulated by chunk copies.  Pooled x0 and scores must be bit-identical to the
unsharded path (P11), and scores within 2e-3 of the oracle."""
import numpy as np
import pytest
import torch

import cvr_synth as cs
import oracle as O
from helpers import TOL_BF16, make_model, to_dev

pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)


@pytest.fixture(scope="module")
def c3small():
    from paper_2605_29232_b200 import build
    build.build()
    cfg = cs.C3.with_(rows=(20000,) * 100)     # config-3 structure (100 fp16 tables x 128, W = 12864)
    tabs = [s.materialize(device="cuda") for s in cs.table_specs(cfg)]
    w = cs.make_weights(cfg)
    ref_model, _, _ = make_model(cfg, max_batch=512, max_nnz=1 << 20, tables=tabs, weights=w)
    return cfg, tabs, w, ref_model


@pytest.mark.parametrize("world", [2, 4, 8])
def test_sharded_matches_unsharded(c3small, world):
    from paper_2605_29232_b200 import CvrModel
    from paper_2605_29232_b200.sharded import local_tables
    cfg, tabs, w, ref = c3small
    B = 256
    Bl = B // world
    bt = cs.make_batch(cfg, 9, batch=B)
    idx, off, dense = to_dev(bt)
    x0_ref = ref.embed(idx, off, B, dense)
    s_ref = ref.dense(x0_ref, B)
    ranks = []
    for r in range(world):
        m = CvrModel(cfg, max_batch=Bl, max_nnz=1 << 20, world_size=world, rank=r)
        lt = local_tables(cfg.n_tables, world, r)
        m.load_tables([tabs[t] for t in lt], lt)
        m.load_weights({k: v.cuda() for k, v in w.items()})
        lb = cs.make_batch(cfg, 9, batch=B, tables=lt)
        sb, rb = m.shard_buffer_bytes(B)
        send = torch.empty(sb, dtype=torch.uint8, device="cuda")
        x0 = m.new_x0(Bl)
        li, lo, _ = to_dev(lb)
        m.embed_shard(li, lo, B, dense[r * Bl:(r + 1) * Bl].contiguous(), send, x0)
        ranks.append((m, send, x0))
    torch.cuda.synchronize()
    for r, (m, send, x0) in enumerate(ranks):
        assert m.status() == 0
        chunk = send.numel() // world
        recv = torch.cat([ranks[s][1][r * chunk:(r + 1) * chunk] for s in range(world)])   # all-to-all
        m.unpack_shard(recv, B, x0)
        s = m.dense(x0, Bl)
        torch.cuda.synchronize()
        assert torch.equal(x0, x0_ref[r * Bl:(r + 1) * Bl]), f"rank {r}: x0 differs"
        assert torch.equal(s, s_ref[r * Bl:(r + 1) * Bl]), f"rank {r}: scores differ"
    ref_scores = O.score_forward(cfg, cs.table_specs(cfg), w, cs.sub_batch(bt, np.arange(0, B, 8)))["scores"]
    assert np.abs(s_ref[::8].double().cpu().numpy() - ref_scores).max() <= TOL_BF16


@pytest.mark.parametrize("world", [2, 4])
def test_fused_exchange_v3_matches_unsharded(c3small, world):
    """V3 with N ranks emulated on one GPU: every rank's gather stores its pooled rows
    straight into the owner's x0 slot through the peer-pointer table and signals the ready flags; the ranks are
    launched in sequence and only then wait (no kernel waits on a later launch), so the flags are already set.
    Four epochs exercise both x0 slots and the free-slot handshake (epochs 3, 4 wait on epochs 1, 2's dense).
    Each rank's x0 and scores must be bit-identical to the unsharded path (P11)."""
    from paper_2605_29232_b200.sharded import FusedShardedScorer, local_tables
    cfg, tabs, w, ref = c3small
    B = 256
    Bl = B // world
    ranks = [FusedShardedScorer(cfg, world, r, B, 1 << 20) for r in range(world)]
    for sc in ranks:
        sc.connect(peers=ranks)
        sc.load_tables([tabs[t] for t in sc.tables])
        sc.load_weights({k: v.cuda() for k, v in w.items()})
    for epoch in (1, 2, 3, 4):
        bt = cs.make_batch(cfg, 13 + epoch, batch=B)
        idx, off, dense = to_dev(bt)
        x0_ref = ref.embed(idx, off, B, dense)
        s_ref = ref.dense(x0_ref, B)
        for r, sc in enumerate(ranks):
            lb = cs.make_batch(cfg, 13 + epoch, batch=B, tables=local_tables(cfg.n_tables, world, r))
            li, lo, _ = to_dev(lb)
            sc.embed(li, lo, dense[r * Bl:(r + 1) * Bl].contiguous())
        for r, sc in enumerate(ranks):
            s = sc.dense()
            torch.cuda.synchronize()
            assert sc.model.status() == 0
            assert sc.epoch == epoch and int(sc.ready.min()) == epoch
            assert torch.equal(sc.x0[epoch % 2], x0_ref[r * Bl:(r + 1) * Bl]), f"epoch {epoch} rank {r}: x0 differs"
            assert torch.equal(s, s_ref[r * Bl:(r + 1) * Bl]), f"epoch {epoch} rank {r}: scores differ"
        assert all(int(sc.free.min()) == epoch for sc in ranks)


def test_sharded_scorer_pipelined_world1(c3small):
    """ShardedScorer's two-stream executor (gather + exchange + unpack of batch k+1 overlapping the dense stage of
    batch k, double-buffered send / recv / x0) at N = 1 (the all-to-all is a local copy): back-to-back batches give
    scores bit-identical to the serial call and to the unsharded path."""
    from paper_2605_29232_b200.sharded import ShardedScorer
    cfg, tabs, w, ref = c3small
    B = 384
    sc = ShardedScorer(cfg, 1, 0, B, 1 << 20)
    sc.load_tables(tabs)
    sc.load_weights({k: v.cuda() for k, v in w.items()})
    batches = [cs.make_batch(cfg, 20 + i, batch=B) for i in range(5)]
    dev_in = [to_dev(bt) for bt in batches]
    refs = [ref.dense(ref.embed(i, o, B, d), B).clone() for i, o, d in dev_in]
    s_e, s_d = torch.cuda.Stream(), torch.cuda.Stream()
    outs = [torch.empty(B, device="cuda") for _ in batches]
    # the side streams do not order after the current stream: the references (and any work on memory the caching
    # allocator just handed back to this stream, e.g. for outs) must be finished first
    torch.cuda.synchronize()
    for (i, o, d), out in zip(dev_in, outs):
        sc.score(i, o, d, out, stream=s_e, s_dense=s_d)
    torch.cuda.synchronize()
    serial = [sc.score(i, o, d).clone() for i, o, d in dev_in]
    torch.cuda.synchronize()
    assert sc.model.status() == 0
    for k, (out, se, r) in enumerate(zip(outs, serial, refs)):
        assert torch.equal(se, r), (k, (se - r).abs().max().item())
        assert torch.equal(out, r), (k, (out - r).abs().max().item())
