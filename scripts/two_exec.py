"""Throughput of E executors (contexts sharing the tables) on one GPU, batches dealt round-robin: does a second
in-flight pipeline fill the SMs the first leaves idle?  (CFG=c2, E=1|2|3; priorities of the dense streams PD)"""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, cvr_synth as cs
from paper_2605_29232_b200 import CvrModel
cfg = cs.CONFIGS[os.environ.get("CFG", "c2")]; B = cfg.batch
NR = 8
ring = [cs.make_batch(cfg, 900 + i) for i in range(NR)]
tabs = [s.materialize(device="cuda") for s in cs.table_specs(cfg)]
w = {k: v.cuda() for k, v in cs.make_weights(cfg).items()}
dev = [(torch.from_numpy(b.indices).cuda(), torch.from_numpy(b.offsets).cuda(), torch.from_numpy(b.dense).cuda()) for b in ring]
outs = [torch.empty(B, device="cuda") for _ in ring]
raw = [(i.data_ptr(), o.data_ptr(), i.numel(), d.data_ptr(), out.data_ptr()) for (i, o, d), out in zip(dev, outs)]
K = int(os.environ.get("K", "600"))
res = {}
for E in [int(x) for x in os.environ.get("E", "1,2").split(",")]:
    ms = []
    for e in range(E):
        m = CvrModel(cfg, max_batch=B, max_nnz=max(b.nnz for b in ring))
        m.load_tables(tabs); m.load_weights(w)
        pr = [int(x) for x in os.environ.get("PRIOS", "0,-1," * E).strip(",").split(",")]
        ms.append((m, torch.cuda.Stream(priority=pr[2 * e]), torch.cuda.Stream(priority=pr[2 * e + 1])))
    def step(i):
        m, se, sd = ms[i % E]
        ip, op, nnz, dp, sp = raw[i % NR]
        m.score_raw(ip, op, nnz, B, dp, sp, se.cuda_stream, sd.cuda_stream)
    for rep in range(3):
        for i in range(40):
            step(i)
        torch.cuda.synchronize()
        a = [torch.cuda.Event(enable_timing=True) for _ in range(E)]
        b = [torch.cuda.Event(enable_timing=True) for _ in range(E)]
        t0 = torch.cuda.Event(enable_timing=True); t0.record()
        torch.cuda.synchronize()
        for e, (m, se, sd) in enumerate(ms):
            se.wait_event(t0); sd.wait_event(t0)
        for i in range(K):
            step(i)
        t1 = torch.cuda.Event(enable_timing=True)
        for e, (m, se, sd) in enumerate(ms):
            ev = torch.cuda.Event(); ev.record(sd); torch.cuda.current_stream().wait_event(ev)
        t1.record(); torch.cuda.synchronize()
        us = t0.elapsed_time(t1) / K * 1e3
        print(json.dumps({"cfg": cfg.name, "executors": E, "rep": rep, "us_per_batch": round(us, 2),
                          "ex_per_s": round(B / us * 1e6)}), flush=True)
    for m, _, _ in ms:
        assert m.status() == 0
    del ms
    torch.cuda.synchronize()
