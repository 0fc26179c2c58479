"""CVR_GEMM_TIMELINE: per-CTA stamps of every GEMM in one dense stage, graph-replayed with PDL as in cvr_score."""
import os, sys, json
os.environ["CVR_GEMM_TIMELINE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, cvr_synth as cs
from paper_2605_29232_b200 import CvrModel
cfg = cs.CONFIGS[os.environ.get("CFG", "c2")]
B = cfg.batch
m = CvrModel(cfg, max_batch=B, max_nnz=1 << 22)
tabs = [s.materialize(device="cuda") for s in cs.table_specs(cfg)]
m.load_tables(tabs); m.load_weights({k: v.cuda() for k, v in cs.make_weights(cfg).items()})
for k, v in (json.loads(sys.argv[1]) if len(sys.argv) > 1 else {}).items():
    m.set_option(k, v)
bt = cs.make_batch(cfg, 0)
idx, off, dense = (torch.from_numpy(bt.indices).cuda(), torch.from_numpy(bt.offsets).cuda(), torch.from_numpy(bt.dense).cuda())
s = torch.cuda.Stream()
x0 = m.embed(idx, off, B, dense, stream=s)
sc = torch.empty(B, device="cuda")
for _ in range(30):
    m.dense(x0, B, sc, stream=s)
torch.cuda.synchronize()
m.close()
