"""A/B the dense stage (graph-replayed) under library options, interleaved to cancel drift."""
import os, sys, json, itertools
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
settings = json.loads(sys.argv[1]) if len(sys.argv) > 1 else [{}, {"pdl": 0}]
K = int(os.environ.get("K", "200"))
res = {i: [] for i in range(len(settings))}
for rep in range(3):
    for i, st in enumerate(settings):
        for k, v in st.items():
            m.set_option(k, v)
        for _ in range(5):
            m.dense(x0, B, sc, stream=s)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(K):
            m.dense(x0, B, sc, stream=s)
        b.record(s); torch.cuda.synchronize()
        res[i].append(a.elapsed_time(b) / K * 1e3)
        for k in st:  # restore defaults
            m.set_option(k, {"pdl": 1, "graphs": 1, "ens_u_bn": 128, "pair": 1, "u_bn": 192, "xv_bn": 0, "epw": 2,
                             "ens_attn_tc": 1, "ens_ffn_fused": 0}.get(k, 1))
roles = [r for r in os.environ.get("ROLES", "").split(",") if r]
for i, st in enumerate(settings):
    out = {"setting": st, "us_per_dense": [round(x, 2) for x in res[i]], "min": round(min(res[i]), 2)}
    for k, v in st.items():
        m.set_option(k, v)
    m.dense(x0, B, sc, stream=s)
    for role in roles:  # per-launch time of one GEMM role in a PDL chain of its own launches (cvr_repeat_kernel)
        n = m.repeat_kernel(role, 4, x0, B, stream=s)
        torch.cuda.synchronize()
        if n == 0:  # this role does not run under this setting
            continue
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(3):
            m.repeat_kernel(role, 4, x0, B, stream=s)
        b.record(s); torch.cuda.synchronize()
        out[role + "_us"] = round(a.elapsed_time(b) * 1e3 / (3 * n), 2)
    for k in st:
        m.set_option(k, {"ens_attn_tc": 1, "ens_ffn_fused": 0}.get(k, 1))
    print(json.dumps(out))
