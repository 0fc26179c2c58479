import os, sys, json, subprocess
sys.path.insert(0, "/root/repo")
import torch, cvr_synth as cs
from paper_2605_29232_b200 import CvrModel
cfg = cs.C2
B = int(os.environ.get("B", "4096"))
m = CvrModel(cfg, max_batch=B, max_nnz=1 << 12)
m.load_weights({k: v.cuda() for k, v in cs.make_weights(cfg).items()})
x0 = m.new_x0(B)
g = torch.Generator(device="cuda").manual_seed(3)
x0[:, :cfg.width] = (torch.randn(B, cfg.width, device="cuda", generator=g) * 0.3).to(x0.dtype)
outs = []
for i in range(3):
    outs.append(m.dense(x0, B).clone())
m.set_option("u_bn", 64)
outs.append(m.dense(x0, B).clone())
torch.save([o.cpu() for o in outs], os.environ["OUT"])
print("saved", [bool(torch.equal(outs[0], o)) for o in outs])
