import os, sys
os.environ["CVR_DEBUG_TIMING"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, cvr_synth as cs
from paper_2605_29232_b200 import CvrModel
cfg = cs.C2
for pdl in (1, 0):
    m = CvrModel(cfg, max_batch=4096, max_nnz=1 << 20)
    tabs = [s.materialize(device="cuda") for s in cs.table_specs(cfg)]
    m.load_tables(tabs); m.load_weights({k: v.cuda() for k, v in cs.make_weights(cfg).items()})
    bt = cs.make_batch(cfg, 0)
    idx, off, dense = (torch.from_numpy(bt.indices).cuda(), torch.from_numpy(bt.offsets).cuda(), torch.from_numpy(bt.dense).cuda())
    x0 = m.embed(idx, off, 4096, dense)
    m.set_option("pdl", pdl)
    m.set_option("fused_cross", 1)
    for _ in range(5):
        s = m.dense(x0, 4096)
    torch.cuda.synchronize()
    print("pdl", pdl, file=sys.stderr)
    m.close()
