"""Serving on the GPU (config 5 machinery): a short open-loop run through the native serving loop (C++ batcher +
host batch assembly + cvr_score_host, libcvr cvr_serve_trace); every served score must be bit-identical to scoring
the same request alone (batching transparency, SPEC.md:672 / SURVEY.md P10), every request must complete, and no
executor graph is captured during the run (all grid-size buckets were captured up front by cvr_warm_graphs).  Also
with two executor lanes (the loop's completion events ride on s_dense, which waits for each lane's work)."""
import numpy as np
import pytest
import torch

import cvr_synth as cs

pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)


@pytest.mark.parametrize("lanes", [1, 2])
def test_served_scores_equal_offline(lanes):
    from paper_2605_29232_b200 import CvrModel, build
    from paper_2605_29232_b200.serving import ItemPoolView, Request, Server
    build.build()
    cfg = cs.C2.with_(rows=(50000,) * 26)
    pool = cs.make_item_pool(cfg, 4096)
    view = ItemPoolView(pool.offsets, pool.indices, pool.dense, cfg.n_tables)
    m = CvrModel(cfg, max_batch=2048, max_nnz=2048 * 26 * 16, lanes=lanes)
    m.load_tables([s.materialize(device="cuda") for s in cs.table_specs(cfg)])
    m.load_weights({k: v.cuda() for k, v in cs.make_weights(cfg).items()})
    trace = cs.make_requests(4000.0, 0.25, 4096, seed=77)
    reqs = [Request(i, t, len(ids), ids) for i, (t, ids) in enumerate(trace)]
    srv = Server(m, view, max_items=2048, window_s=0.002, max_nnz=2048 * 26 * 16)
    captured = m.call_info(0)["graph_captures"]
    from paper_2605_29232_b200._cvr import EXECUTOR_SLOTS as NS
    assert captured == lanes * NS * 2 * 5  # lanes x slots x (embed, dense) x buckets 128 .. 2048
    lat, sizes, scores = srv.run(reqs, keep_scores=True)
    assert m.call_info(0)["graph_captures"] == captured
    assert srv.stats["rejected"] == 0 and not srv.stats["aborted"]
    assert np.all(np.isfinite(lat)) and sizes.sum() == sum(r.n_items for r in reqs)
    assert sizes.max() <= 2048
    for r in reqs[:: max(1, len(reqs) // 12)]:
        sub = cs.sub_batch(pool, r.item_ids)
        idx, off, dense = (torch.from_numpy(sub.indices).cuda(), torch.from_numpy(sub.offsets).cuda(),
                           torch.from_numpy(sub.dense).cuda())
        offline = m.dense(m.embed(idx, off, r.n_items, dense), r.n_items).cpu().numpy()
        assert np.array_equal(offline, scores[r.rid])
