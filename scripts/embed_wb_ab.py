"""A/B the warp-per-bag gather (option embed_wb) against the lane-group-per-bag kernel on config 2 (or CFG):
isolated embedding stage, pipelined executor step, and the pooled x0 difference."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np, cvr_synth as cs
import bench
from paper_2605_29232_b200 import CvrModel
cfg = cs.CONFIGS[os.environ.get("CFG", "c2")]
B = cfg.batch
m = CvrModel(cfg, max_batch=B, max_nnz=1 << 23)
tabs = [s.materialize(device="cuda") for s in cs.table_specs(cfg)]
m.load_tables(tabs); m.load_weights({k: v.cuda() for k, v in cs.make_weights(cfg).items()})
ring = [cs.make_batch(cfg, 700 + i) for i in range(8)]
dev = [(torch.from_numpy(b.indices).cuda(), torch.from_numpy(b.offsets).cuda(), torch.from_numpy(b.dense).cuda()) for b in ring]
outs = [torch.empty(B, device="cuda") for _ in ring]
byts = float(np.mean([bench.embed_bytes(cfg, b) for b in ring]))
s_e, s_d = torch.cuda.Stream(), torch.cuda.Stream(priority=-1)
x0a, x0b = m.new_x0(B), m.new_x0(B)
m.embed(*dev[0][:2], B, dev[0][2], x0=x0a); m.set_option("embed_wb", 1); m.embed(*dev[0][:2], B, dev[0][2], x0=x0b)
m.set_option("embed_wb", 0); torch.cuda.synchronize()
d = (x0a.float() - x0b.float()).abs().max().item()
print(json.dumps({"x0_max_abs_diff_wb_vs_default": d}), flush=True)
for rep in range(3):
    for wb in (0, 1):
        m.set_option("embed_wb", wb)
        def run(i):
            m.embed(*dev[i % 8][:2], B, dev[i % 8][2], x0=x0a, stream=s_e)
        for i in range(8): run(i)
        torch.cuda.synchronize()
        us = bench.time_enqueued(run, 200, s_e) * 1e3
        for i in range(20):
            m.score(*dev[i % 8][:2], B, dev[i % 8][2], outs[i % 8], s_embed=s_e, s_dense=s_d)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s_e); s_d.wait_event(e0)
        for i in range(200):
            m.score(*dev[i % 8][:2], B, dev[i % 8][2], outs[i % 8], s_embed=s_e, s_dense=s_d)
        e1.record(s_d); torch.cuda.synchronize()
        print(json.dumps({"wb": wb, "embed_us": round(us, 2), "frac_hbm": round(byts / us / 1e3 / 6556.8, 3),
                          "step_us": round(e0.elapsed_time(e1) / 200 * 1e3, 2)}), flush=True)
assert m.status(s_d) == 0
