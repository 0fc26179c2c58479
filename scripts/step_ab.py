"""A/B the pipelined cvr_score step under executor / kernel options, interleaved (CFG=c2|c3s|c4|c6)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, cvr_synth as cs
from paper_2605_29232_b200 import CvrModel
cfg = cs.CONFIGS[os.environ.get("CFG", "c2")]; B = cfg.batch
NR = int(os.environ.get("RING", "8"))
ring = [cs.make_batch(cfg, 900 + i) for i in range(NR)]
m = CvrModel(cfg, max_batch=B, max_nnz=max(b.nnz for b in ring), lanes=int(os.environ.get("LANES", "1")))
tabs = [s.materialize(device="cuda") for s in cs.table_specs(cfg)]
m.load_tables(tabs); m.load_weights({k: v.cuda() for k, v in cs.make_weights(cfg).items()})
dev = [(torch.from_numpy(b.indices).cuda(), torch.from_numpy(b.offsets).cuda(), torch.from_numpy(b.dense).cuda()) for b in ring]
outs = [torch.empty(B, device="cuda") for _ in ring]
PE, PD = (int(x) for x in os.environ.get("PRIO", "0,-1").split(","))  # stream priorities (lower = higher)
se, sd = torch.cuda.Stream(priority=PE), torch.cuda.Stream(priority=PD)
raw = [(i.data_ptr(), o.data_ptr(), i.numel(), d.data_ptr(), out.data_ptr()) for (i, o, d), out in zip(dev, outs)]
settings = json.loads(sys.argv[1])
K = int(os.environ.get("K", "500"))
DEF = {"u_bn": 192, "epw": 0, "pdl": 1, "graphs": 1, "embed_bps": 0, "xv_bn": 0, "prefetch_b": 1,
       "ens_fused_attn": 1, "zero_copy_scores": 1, "ens_ffn_fused": 0}  # (restored after each setting; others -> 1)
for rep in range(3):
    for st in settings:
        for k, v in st.items(): m.set_option(k, v)
        for i in range(20):
            ip, op, nnz, dp, sp = raw[i % NR]; m.score_raw(ip, op, nnz, B, dp, sp, se.cuda_stream, sd.cuda_stream)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(se); sd.wait_event(a)
        for i in range(K):
            ip, op, nnz, dp, sp = raw[i % NR]; m.score_raw(ip, op, nnz, B, dp, sp, se.cuda_stream, sd.cuda_stream)
        b.record(sd); torch.cuda.synchronize()
        print(json.dumps({"cfg": cfg.name, "rep": rep, "setting": st, "us_per_step": round(a.elapsed_time(b) / K * 1e3, 2)}), flush=True)
        for k in st: m.set_option(k, DEF.get(k, 1))
