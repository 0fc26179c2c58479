"""Probe: cvr_score throughput with L executor lanes (L contexts sharing the tables, each with its own embed /
dense streams), batches round-robin over lanes.  L = 1 is bench.py's executor."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, cvr_synth as cs
from paper_2605_29232_b200 import CvrModel

cfg = cs.CONFIGS[os.environ.get("CFG", "c2")]
B = cfg.batch
dev = torch.device("cuda", 0)
tables = [s.materialize(device=dev) for s in cs.table_specs(cfg)]
w = {k: v.to(dev) for k, v in cs.make_weights(cfg).items()}
ring = [cs.make_batch(cfg, 1000 + i) for i in range(8)]
max_nnz = max(b.nnz for b in ring)
dev_in = [(torch.from_numpy(b.indices).to(dev), torch.from_numpy(b.offsets).to(dev), torch.from_numpy(b.dense).to(dev))
          for b in ring]
outs = [torch.empty(B, device=dev) for _ in ring]
ms = []
for _ in range(2):
    m = CvrModel(cfg, max_batch=B, max_nnz=max_nnz, device=dev)
    m.load_tables(tables); m.load_weights(w)
    ms.append(m)
streams = [(torch.cuda.Stream(dev, priority=0), torch.cuda.Stream(dev, priority=-1)) for _ in range(2)]
K = int(os.environ.get("K", "1000"))


def run(L, k):
    for i in range(k):
        j = i % L
        idx, off, dn = dev_in[i % 8]
        ms[j].score(idx, off, B, dn, outs[i % 8], s_embed=streams[j][0], s_dense=streams[j][1])


res = {}
for rep in range(3):
    for L in (1, 2):
        run(L, 20); torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(streams[0][0])
        for se, sd in streams:
            se.wait_event(a); sd.wait_event(a)
        run(L, K)
        for se, sd in streams:
            e = torch.cuda.Event(); e.record(sd); streams[0][0].wait_event(e)
        b.record(streams[0][0]); torch.cuda.synchronize()
        us = a.elapsed_time(b) / K * 1e3
        res.setdefault(L, []).append(round(us, 2))
for L, v in res.items():
    print(json.dumps({"lanes": L, "us_per_step": v, "examples_per_s": round(B / (min(v) * 1e-6))}))
