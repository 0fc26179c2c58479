"""Per-role kernel times of the dense stage (CUDA-event pair around every launch) under option settings."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, cvr_synth as cs
from paper_2605_29232_b200 import CvrModel

cfg = cs.CONFIGS[os.environ.get("CFG", "c2")]
B = cfg.batch
m = CvrModel(cfg, max_batch=B, max_nnz=1 << 22)
tabs = [s.materialize(device="cuda") for s in cs.table_specs(cfg)]
m.load_tables(tabs); m.load_weights({k: v.cuda() for k, v in cs.make_weights(cfg).items()})
bt = cs.make_batch(cfg, 0)
idx, off, dense = (torch.from_numpy(bt.indices).cuda(), torch.from_numpy(bt.offsets).cuda(), torch.from_numpy(bt.dense).cuda())
s = torch.cuda.Stream()
x0 = m.embed(idx, off, B, dense, stream=s)
sc = torch.empty(B, device="cuda")
settings = json.loads(sys.argv[1]) if len(sys.argv) > 1 else [{}]
for st in settings:
    for k, v in st.items():
        m.set_option(k, v)
    for _ in range(5):
        m.dense(x0, B, sc, stream=s)
    torch.cuda.synchronize()
    m.profile_begin(4000)
    for _ in range(int(os.environ.get("K", "100"))):
        m.dense(x0, B, sc, stream=s)
    torch.cuda.synchronize()
    prof = m.profile_end()
    print(json.dumps({"setting": st, "kernels": {k: round(v["avg_ms"] * 1e3, 2) for k, v in prof.items()},
                      "launches": {k: v["launches"] for k, v in prof.items()}}))
    for k in st:
        m.set_option(k, {"pdl": 1, "graphs": 1, "u_bn": 192, "xv_bn": 0, "epw": 2}.get(k, 1))
