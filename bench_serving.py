#!/usr/bin/env python
"""Config 5 (BASELINE.json configs[4]): serving with dynamic batching.

Poisson request arrivals at {2k, 8k, 32k} queries/s (open loop, seeded), items per query
lognormal(mu=ln 50, sigma=0.8) capped at 500 drawn from a seeded pool of config-2 items; server-side
dynamic batching (max 8192 items, 2 ms window anchored at the oldest request), host batch assembly into
pinned staging (libcvr cvr_gather_items), decoupled execution through cvr_score_host (copy stream ->
embed stream -> dense stream -> D2H).  Reports p50/p99 latency (nearest rank, from the scheduled
arrival), served queries/s and items/s, batch-size statistics, and checks a sample of served scores
bit-exactly against the same items scored offline (batching transparency).

    python bench_serving.py [--qps 2000 8000 32000] [--duration 2.0] [--window-ms 2.0]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import cvr_synth as cs  # noqa: E402
from paper_2605_29232_b200 import CvrModel  # noqa: E402
from paper_2605_29232_b200.serving import ItemPoolView, Request, Server, nearest_rank  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--qps", type=float, nargs="+", default=[2000.0, 8000.0, 32000.0])
    ap.add_argument("--duration", type=float, default=2.0)
    ap.add_argument("--warmup", type=float, default=0.3)
    ap.add_argument("--window-ms", type=float, default=2.0)
    ap.add_argument("--max-items", type=int, default=8192)
    ap.add_argument("--pool", type=int, default=1 << 16)
    args = ap.parse_args()
    cfg = cs.C2
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", "0")))
    pool = cs.make_item_pool(cfg, args.pool)
    view = ItemPoolView(pool.offsets, pool.indices, pool.dense, cfg.n_tables)
    item_nnz = np.diff(pool.offsets).reshape(cfg.n_tables, args.pool).sum(axis=0)
    max_nnz = int(np.sort(item_nnz)[-args.max_items:].sum())
    m = CvrModel(cfg, max_batch=args.max_items, max_nnz=max_nnz, device=dev)
    tables = [s.materialize(device=dev) for s in cs.table_specs(cfg)]
    m.load_tables(tables)
    m.load_weights({k: v.to(dev) for k, v in cs.make_weights(cfg).items()})
    results = []
    for qps in args.qps:
        trace = cs.make_requests(qps, args.warmup + args.duration, args.pool)
        reqs = [Request(i, t, len(ids), ids) for i, (t, ids) in enumerate(trace)]
        srv = Server(m, view, max_items=args.max_items, window_s=args.window_ms / 1e3, max_nnz=max_nnz)
        lat, sizes, scores = srv.run(reqs, keep_scores=True)
        meas = [r.rid for r in reqs if r.t_arrival >= args.warmup]
        L = lat[meas] * 1e3
        n_items = sum(reqs[i].n_items for i in meas)
        # batching transparency: re-score 16 served requests offline (one batch each) -> bit-equal
        chk = meas[:: max(1, len(meas) // 16)][:16]
        ok = True
        for rid in chk:
            ids = reqs[rid].item_ids
            sub = cs.sub_batch(pool, ids)
            idx, off, dense = (torch.from_numpy(sub.indices).to(dev), torch.from_numpy(sub.offsets).to(dev),
                               torch.from_numpy(sub.dense).to(dev))
            s_off = m.dense(m.embed(idx, off, len(ids), dense), len(ids)).cpu().numpy()
            ok &= bool(np.array_equal(s_off, scores[rid]))
        res = {"qps_offered": qps, "queries": len(meas), "items": int(n_items),
               "p50_ms": float(nearest_rank(L, 50)), "p99_ms": float(nearest_rank(L, 99)),
               "mean_ms": float(np.mean(L)), "served_items_per_s": n_items / args.duration,
               "batches": int(len(sizes)), "batch_items_mean": float(sizes.mean()), "batch_items_max": int(sizes.max()),
               "rejected": int(srv.batcher.rejected), "transparency_bitexact": ok, "checked_requests": len(chk)}
        results.append(res)
        print(json.dumps(res), flush=True)
    print(json.dumps({"metric": "p50/p99 latency under dynamic batching (config 5)", "window_ms": args.window_ms,
                      "max_items": args.max_items, "pool": args.pool, "duration_s": args.duration,
                      "results": results}), flush=True)


if __name__ == "__main__":
    main()
