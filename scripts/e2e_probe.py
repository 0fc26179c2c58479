"""Probe the host-fed (e2e) step: device-resident cvr_score vs cvr_score_host vs the H2D copies alone."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, cvr_synth as cs
from paper_2605_29232_b200 import CvrModel

cfg = cs.CONFIGS[os.environ.get("CFG", "c2")]
B = cfg.batch
dev = torch.device("cuda", 0)
tables = [s.materialize(device=dev) for s in cs.table_specs(cfg)]
ring = [cs.make_batch(cfg, 1000 + i) for i in range(8)]
m = CvrModel(cfg, max_batch=B, max_nnz=max(b.nnz for b in ring), device=dev)
m.load_tables(tables); m.load_weights({k: v.to(dev) for k, v in cs.make_weights(cfg).items()})
host = [(torch.from_numpy(b.indices).pin_memory(), torch.from_numpy(b.offsets).pin_memory(),
         torch.from_numpy(b.dense).pin_memory()) for b in ring]
devin = [tuple(t.to(dev) for t in h) for h in host]
hout = [torch.empty(B).pin_memory() for _ in ring]
dout = [torch.empty(B, device=dev) for _ in ring]
s_c, s_e, s_d = torch.cuda.Stream(dev), torch.cuda.Stream(dev), torch.cuda.Stream(dev, priority=-1)
dst = [tuple(torch.empty_like(t, device=dev) for t in h) for h in host]
K = int(os.environ.get("K", "500"))


def timed(fn, first, last):
    for i in range(20):
        fn(i)
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(first)
    for s in (s_c, s_e, s_d):
        s.wait_event(a)
    for i in range(K):
        fn(i)
    for s in (s_c, s_e, s_d, s_r):
        e = torch.cuda.Event(); e.record(s); last.wait_event(e)
    b.record(last); torch.cuda.synchronize()
    return a.elapsed_time(b) / K * 1e3


def dev_step(i):
    idx, off, dn = devin[i % 8]
    m.score(idx, off, B, dn, dout[i % 8], s_embed=s_e, s_dense=s_d)


s_r = torch.cuda.Stream(dev)


def dev_d2h_step(i):  # + D2H of the scores on the dense stream
    dev_step(i)
    with torch.cuda.stream(s_d):
        hout[i % 8].copy_(dout[i % 8], non_blocking=True)


def dev_d2h_side_step(i):  # + D2H on a side stream after an event
    dev_step(i)
    e = torch.cuda.Event(); e.record(s_d); s_r.wait_event(e)
    with torch.cuda.stream(s_r):
        hout[i % 8].copy_(dout[i % 8], non_blocking=True)


def dev_h2d_step(i):  # device-resident scoring + unrelated H2D traffic of the same size on the copy stream
    dev_step(i)
    copy_step(i)


def host_step(i):
    idx, off, dn = host[i % 8]
    m.score_host(idx, off, B, dn, hout[i % 8], s_copy=s_c, s_embed=s_e, s_dense=s_d)


def copy_step(i):
    with torch.cuda.stream(s_c):
        for d, h in zip(dst[i % 8], host[i % 8]):
            d.copy_(h, non_blocking=True)


res = {}
for rep in range(3):
    for name, fn in (("device_score", dev_step), ("host_score", host_step), ("h2d_only", copy_step),
                     ("device+d2h", dev_d2h_step), ("device+d2h_side", dev_d2h_side_step), ("device+h2d", dev_h2d_step)):
        res.setdefault(name, []).append(round(timed(fn, s_c, s_c), 2))
nbytes = sum(t.numel() * t.element_size() for t in host[0])
for k, v in res.items():
    print(json.dumps({"probe": k, "us_per_step": v, "h2d_bytes": nbytes}))
