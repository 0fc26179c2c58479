"""Probe: the library's own NCCL communicator at world 1 (cvr_comm_unique_id -> cvr_comm_init)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import cvr_synth as cs
from paper_2605_29232_b200 import CvrModel
from paper_2605_29232_b200._cvr import comm_unique_id
torch.cuda.set_device(0)
cfg = cs.C3.with_(rows=(2000,) * 100)
m = CvrModel(cfg, max_batch=64, max_nnz=1 << 16, world_size=1, rank=0)
uid = comm_unique_id()
print("uid", uid[:16].hex(), flush=True)
m.comm_init(uid, 1, 0)
print("comm_init ok", flush=True)
