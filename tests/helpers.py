"""Shared test plumbing: build a CvrModel from a cvr_synth config, slice batches (CSR index
arithmetic only), and the tolerances of BASELINE.json's north star."""
from __future__ import annotations

import numpy as np
import torch

import cvr_synth as cs
from cvr_synth import sub_batch  # noqa: F401

TOL_F32 = 1e-5   # BASELINE.json north star: fp32 path, absolute on scores
TOL_BF16 = 2e-3  # BASELINE.json north star: bf16 path, absolute on the sigmoid output


def device_tables(cfg, device="cuda"):
    return [spec.materialize(device=device) for spec in cs.table_specs(cfg)]


def to_dev(bt: cs.Batch, device="cuda"):
    return (torch.from_numpy(bt.indices).to(device), torch.from_numpy(bt.offsets).to(device),
            torch.from_numpy(bt.dense).to(device))


def make_model(cfg, max_batch, max_nnz=0, tables=None, weights=None, device="cuda", lanes=1):
    from paper_2605_29232_b200 import CvrModel
    m = CvrModel(cfg, max_batch=max_batch, max_nnz=max_nnz, device=device, lanes=lanes)
    tables = device_tables(cfg, device) if tables is None else tables
    m.load_tables(tables)
    w = cs.make_weights(cfg) if weights is None else weights
    m.load_weights({k: v.to(device) for k, v in w.items()})
    return m, tables, w
