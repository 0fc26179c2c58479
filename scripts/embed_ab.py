"""Time the embedding stage alone (IDX=uniform: the uniform-index control); reports us and GB/s on algorithmic
and compulsory (distinct rows once) bytes."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, cvr_synth as cs
from paper_2605_29232_b200 import CvrModel
cfg = cs.CONFIGS[os.environ.get("CFG", "c2")]
B = cfg.batch
m = CvrModel(cfg, max_batch=B, max_nnz=1 << 23)
tabs = [s.materialize(device="cuda") for s in cs.table_specs(cfg)]
m.load_tables(tabs); m.load_weights({k: v.cuda() for k, v in cs.make_weights(cfg).items()})
ring = [cs.make_batch(cfg, 700 + i, index_mode=os.environ.get("IDX")) for i in range(4)]
dev = [(torch.from_numpy(b.indices).cuda(), torch.from_numpy(b.offsets).cuda(), torch.from_numpy(b.dense).cuda()) for b in ring]
row = cfg.dim * (4 if cfg.emb_dtype == "f32" else 2); act = 4 if cfg.act_dtype == "f32" else 2
byts = sum(b.nnz * (row + 4) + (cfg.n_tables * B + 1) * 4 + B * cfg.n_tables * cfg.dim * act + B * cfg.n_dense * (4 + act) for b in ring) / len(ring)
import numpy as np


def distinct_rows(b):  # compulsory traffic: every distinct (table, row) once
    offs = b.offsets.astype(np.int64)
    return sum(len(np.unique(b.indices[offs[t * B]:offs[(t + 1) * B]])) for t in range(cfg.n_tables))


cbyts = sum(distinct_rows(b) * row + b.nnz * 4 + (cfg.n_tables * B + 1) * 4 + B * cfg.n_tables * cfg.dim * act
            + B * cfg.n_dense * (4 + act) for b in ring) / len(ring)
s = torch.cuda.Stream()
x0 = m.new_x0(B)
K = 200
settings = json.loads(sys.argv[1]) if len(sys.argv) > 1 else [{}]
for rep in range(3):
    for v2 in settings:
        for k, v in v2.items():
            m.set_option(k, v)
        for i in range(8):
            m.embed(*dev[i % 4][:2], B, dev[i % 4][2], x0=x0, stream=s)
        torch.cuda.synchronize()
        import bench
        us = bench.time_enqueued(lambda i: m.embed(*dev[i % 4][:2], B, dev[i % 4][2], x0=x0, stream=s), K, s) * 1e3
        print(json.dumps({"cfg": cfg.name, "index_mode": os.environ.get("IDX") or cfg.zipf_mode, "variant": v2,
                          "us": round(us, 2), "GBps_alg": round(byts / us / 1e3, 1),
                          "frac_hbm": round(byts / us / 1e3 / 6556.5, 3),
                          "frac_hbm_compulsory": round(cbyts / us / 1e3 / 6556.5, 3)}))
        for k in v2:  # (every option this script varies defaults to 0)
            m.set_option(k, 0)
assert m.status(s) == 0
