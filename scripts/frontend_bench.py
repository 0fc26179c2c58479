"""Feature front end on B200: the hashed gather (cvr_embed_keys: FNV-1a + mean pooling
fused into the embedding kernel) vs the row-id gather (cvr_embed) on the SAME bags (row ids = the oracle's
hash of the keys), and the full pipelined cvr_score_keys step, config c7 (c2 model, B = 4096).
Writes one JSON line (stdout)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import cvr_synth as cs
import oracle as O
from paper_2605_29232_b200 import CvrModel, frontend as F

cfg, spec = cs.C7, cs.FRONTEND_C7
B = cfg.batch
fbs = [cs.make_feature_batch(cfg, i, batch=B) for i in range(4)]
ring = [F.assemble_keys(fb, spec) for fb in fbs]
rows = []
for fb in fbs[:1]:
    r, o, modes = O.frontend_rows(cfg, fb, spec)   # row ids for the same bags (the index-mode comparison)
    rows.append((r.astype(np.int32), o.astype(np.int32)))
m = CvrModel(cfg, max_batch=B, max_nnz=max(len(k) for k, _ in ring))
tabs = [s.materialize(device="cuda") for s in cs.table_specs(cfg)]
m.load_tables(tabs)
m.load_weights({k: v.cuda() for k, v in cs.make_weights(cfg).items()})
vocab, mode = F.feature_spec(cfg, spec)
m.set_feature_spec(vocab, mode)
dev = [(torch.from_numpy(k).cuda(), torch.from_numpy(o).cuda(), torch.from_numpy(fb.dense).cuda())
       for (k, o), fb in zip(ring, fbs)]
idx0 = (torch.from_numpy(rows[0][0]).cuda(), torch.from_numpy(rows[0][1]).cuda())
x0 = m.new_x0(B)
s = torch.cuda.Stream()


def timed(fn, n=200):
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(n):
        fn()
    b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n * 1e3


k0, o0, d0 = dev[0]
t_keys = timed(lambda: m.embed_keys(k0, o0, B, d0, x0=x0, stream=s))
t_rows = timed(lambda: m.embed(idx0[0], idx0[1], B, d0, x0=x0, stream=s))
outs = [torch.empty(B, device="cuda") for _ in dev]
se, sd = torch.cuda.Stream(priority=0), torch.cuda.Stream(priority=-1)
for i in range(20):
    k, o, d = dev[i % 4]
    m.score_keys(k, o, B, d, scores=outs[i % 4], s_embed=se, s_dense=sd)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(se)
sd.wait_event(a)
N = 500
for i in range(N):
    k, o, d = dev[i % 4]
    m.score_keys(k, o, B, d, scores=outs[i % 4], s_embed=se, s_dense=sd)
b.record(sd)
torch.cuda.synchronize()
step_us = a.elapsed_time(b) / N * 1e3
assert m.status() == 0
nnz = len(ring[0][0])
print(json.dumps({"workload": "c7: config-2 model on raw features (20 categorical key tables, 3 text 3-gram tables, "
                              "3 history tables truncated to 50; FNV-1a hashed, text/history mean-pooled)",
                  "batch": B, "nnz": nnz, "embed_keys_us": round(t_keys, 2), "embed_rowids_us": round(t_rows, 2),
                  "hash_overhead_pct": round(100 * (t_keys / t_rows - 1), 1),
                  "score_keys_step_us": round(step_us, 2), "examples_per_s": B / step_us * 1e6}))
m.close()
