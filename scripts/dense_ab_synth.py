"""A/B the dense stage on a synthetic x0 (no tables: large configs without materialising them), options
interleaved to cancel drift.  CFG=c3s B=65536 python scripts/dense_ab_synth.py '[{}, {"xv_bn": 256}]'"""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, cvr_synth as cs
from paper_2605_29232_b200 import CvrModel

cfg = cs.CONFIGS[os.environ.get("CFG", "c2")]
B = int(os.environ.get("B", cfg.batch))
m = CvrModel(cfg, max_batch=B, max_nnz=1 << 12)
m.load_weights({k: v.cuda() for k, v in cs.make_weights(cfg).items()})
x0 = m.new_x0(B)
g = torch.Generator(device="cuda").manual_seed(0)
W = cfg.n_tables * cfg.dim + cfg.n_dense
x0[:, :W] = (torch.randn(B, W, device="cuda", generator=g) * 0.3).to(x0.dtype)
s = torch.cuda.Stream()
sc = torch.empty(B, device="cuda")
settings = json.loads(sys.argv[1]) if len(sys.argv) > 1 else [{}]
K = int(os.environ.get("K", "20"))
defaults = {"a_resident": 0, "pdl": 1, "fused_cross": 0, "graphs": 1, "stack": 0, "ens_u_bn": 128, "pair": 1,
            "u_bn": 192, "mc": 0, "mb": 0, "pair_mlp": 0, "pair_xv": 0, "xv_bn": 0, "xv_splitk": 0, "prefetch_b": 1, "pair_u": 0, "ens_fused_attn": 1, "ens_attn_ar": 0, "f32_tma_store": 1}
res = {i: [] for i in range(len(settings))}
ref = None
for rep in range(3):
    for i, st in enumerate(settings):
        for k, v in st.items():
            m.set_option(k, v)
        for _ in range(3):
            m.dense(x0, B, sc, stream=s)
        torch.cuda.synchronize()
        if ref is None:
            ref = sc.clone()
        same = bool(torch.equal(sc, ref))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(K):
            m.dense(x0, B, sc, stream=s)
        b.record(s); torch.cuda.synchronize()
        res[i].append((a.elapsed_time(b) / K * 1e3, same))
        for k in st:
            m.set_option(k, defaults.get(k, 1))
for i, st in enumerate(settings):
    print(json.dumps({"cfg": cfg.name, "B": B, "setting": st, "us_per_dense": [round(x, 2) for x, _ in res[i]],
                      "min": round(min(x for x, _ in res[i]), 2), "bit_equal_to_first": all(e for _, e in res[i])}))
