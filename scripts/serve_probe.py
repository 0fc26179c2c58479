"""Probe the native serving loop's per-batch costs: host dispatch time per batch (cvr_serve_stats), the executor's
device time for one small batch (cvr_score_host back to back, CUDA events), and the no-batching service rate."""
import os, sys, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import cvr_synth as cs
from paper_2605_29232_b200 import CvrModel
from paper_2605_29232_b200.serving import ItemPoolView, Server, nearest_rank
cfg = cs.C2
dev = torch.device("cuda", 0)
pool_n = 1 << 16
pool = cs.make_item_pool(cfg, pool_n)
view = ItemPoolView(pool.offsets, pool.indices, pool.dense, cfg.n_tables)
item_nnz = np.diff(pool.offsets).reshape(cfg.n_tables, pool_n).sum(axis=0)
max_nnz = int(np.sort(item_nnz)[-8192:].sum())
m = CvrModel(cfg, max_batch=8192, max_nnz=max_nnz, device=dev)
m.load_tables([s.materialize(device=dev) for s in cs.table_specs(cfg)])
m.load_weights({k: v.to(dev) for k, v in cs.make_weights(cfg).items()})
# device time of back-to-back small batches through cvr_score_host
for B in (68, 512, 4096):
    bt = cs.sub_batch(pool, np.arange(B))
    hi = [torch.from_numpy(bt.indices).pin_memory(), torch.from_numpy(bt.offsets).pin_memory(),
          torch.from_numpy(bt.dense).pin_memory()]
    ho = [torch.empty(B).pin_memory() for _ in range(4)]
    sc, se, sd = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream(priority=-1)
    for i in range(10):
        m.score_host(hi[0], hi[1], B, hi[2], ho[i % 4], s_copy=sc, s_embed=se, s_dense=sd)
    torch.cuda.synchronize()
    n = 200
    t0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(sc); se.wait_event(e0); sd.wait_event(e0)
    for i in range(n):
        m.score_host(hi[0], hi[1], B, hi[2], ho[i % 4], s_copy=sc, s_embed=se, s_dense=sd)
    e1.record(sd)
    t_host = (time.perf_counter() - t0) / n
    torch.cuda.synchronize()
    print(json.dumps({"B": B, "device_us_per_batch": e0.elapsed_time(e1) / n * 1e3, "host_enqueue_us": t_host * 1e6}), flush=True)
for window, qps, mr in [(0.0, 2000.0, 1), (0.0, 10000.0, 1), (0.5e-3, 500.0, 0), (4e-3, 500.0, 0), (0.5e-3, 500.0, 0),
                        (4e-3, 500.0, 0), (1e-3, 200000.0, 0), (1e-3, 300000.0, 0)]:
    t, nn, start, ids = cs.make_requests_flat(qps, 3.0 if qps < 1e4 else 1.0, pool_n)
    srv = Server(m, view, max_items=8192, window_s=window, max_nnz=max_nnz, max_requests=mr or None)
    lat, sizes, _ = srv.run_arrays(t, nn, start, ids, abort_after_s=0.05)
    meas = t >= 0.3
    st = srv.stats
    L = lat[meas]
    worst = np.argsort(-np.where(np.isfinite(lat), lat, 1e9))[:5]
    print(json.dumps({"window_ms": window * 1e3, "qps": qps, "p50_ms": float(nearest_rank(L, 50)) * 1e3,
                      "p99_ms": float(nearest_rank(L, 99)) * 1e3, "max_ms": float(np.max(L)) * 1e3,
                      "batches": int(len(sizes)), "host_dispatch_us_per_batch": st["host_dispatch_s"] / max(1, len(sizes)) * 1e6,
                      "max_dispatch_ms": st["max_dispatch_s"] * 1e3, "max_gather_ms": st["max_gather_s"] * 1e3, "loop_gaps_1ms": st["loop_gaps_1ms"],
                      "aborted": st["aborted"], "worst_at_s": [round(float(t[i]), 4) for i in worst]}), flush=True)
