"""Probe: do two dense stages on two streams (two contexts, batches k and k+1) fill each other's GEMM fill /
drain gaps?  Prints us per dense stage (aggregate) for 1 stream vs 2 concurrent streams, PDL on / off."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, cvr_synth as cs
from paper_2605_29232_b200 import CvrModel

cfg = cs.CONFIGS[os.environ.get("CFG", "c2")]
B = cfg.batch
tabs = [s.materialize(device="cuda") for s in cs.table_specs(cfg)]
w = {k: v.cuda() for k, v in cs.make_weights(cfg).items()}
ms = []
for _ in range(2):
    m = CvrModel(cfg, max_batch=B, max_nnz=1 << 22)
    m.load_tables(tabs); m.load_weights(w)
    ms.append(m)
bt = cs.make_batch(cfg, 0)
idx, off, dense = (torch.from_numpy(bt.indices).cuda(), torch.from_numpy(bt.offsets).cuda(), torch.from_numpy(bt.dense).cuda())
ss = [torch.cuda.Stream(), torch.cuda.Stream()]
x0s = [ms[i].embed(idx, off, B, dense, stream=ss[i]) for i in range(2)]
scs = [torch.empty(B, device="cuda") for _ in range(2)]
K = int(os.environ.get("K", "400"))


def run(nstreams, k):
    for j in range(k):
        i = j % nstreams
        ms[i].dense(x0s[i], B, scs[i], stream=ss[i])


res = {}
for rep in range(3):
    for pdl in (1, 0):
        for m in ms:
            m.set_option("pdl", pdl)
        for ns in (1, 2):
            run(ns, 8); torch.cuda.synchronize()
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            a.record(ss[0])
            for s in ss[1:]:
                s.wait_event(a)
            run(ns, K)
            for s in ss[1:]:
                e = torch.cuda.Event(); e.record(s); ss[0].wait_event(e)
            b.record(ss[0]); torch.cuda.synchronize()
            res.setdefault(f"pdl{pdl}_streams{ns}", []).append(round(a.elapsed_time(b) / K * 1e3, 2))
for k, v in res.items():
    print(json.dumps({"setting": k, "us_per_dense": v, "min": min(v)}))
