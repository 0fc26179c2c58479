"""Sharding simulator -- TEST INFRASTRUCTURE ONLY (see oracle/__init__).

Pure index arithmetic for table-wise sharding (BASELINE.json configs[2]):
table t lives on rank t mod N in slot t div N; rank s sends to rank d the pooled rows of d's batch slice
[d*B/N, (d+1)*B/N) for s's tables, laid out destination-major send[s][d][b_local][slot][:]; the
all-to-all delivers recv[d][s] = send[s][d]; unpacking puts recv[d][s][b][slot] at canonical x0 column
block t = slot*N + s of local row b.  Reassembling every rank's slice must reproduce the canonical
concatenation (tables in id order) exactly -- the exchange is a copy (P11).
"""
from __future__ import annotations

import numpy as np


def owner(t: int, world: int) -> int:
    return t % world


def slot(t: int, world: int) -> int:
    return t // world


def n_slots(n_tables: int, world: int) -> int:
    return (n_tables + world - 1) // world


def build_send(pooled: np.ndarray, world: int, src: int) -> np.ndarray:
    """pooled: [B, T, d] (all tables, global batch) -> rank src's send buffer [N, B/N, S, d]
    (slots of tables src does not own stay 0)."""
    B, T, d = pooled.shape
    Bl, S = B // world, n_slots(T, world)
    send = np.zeros((world, Bl, S, d), dtype=pooled.dtype)
    for t in range(T):
        if owner(t, world) != src:
            continue
        for dst in range(world):
            send[dst, :, slot(t, world), :] = pooled[dst * Bl:(dst + 1) * Bl, t, :]
    return send


def all_to_all(sends):
    """recv[d][s] = send[s][d]."""
    world = len(sends)
    return [np.stack([sends[s][d] for s in range(world)]) for d in range(world)]


def unpack(recv: np.ndarray, n_tables: int, world: int) -> np.ndarray:
    """recv [N(src), B/N, S, d] -> pooled columns of the local slice in canonical order [B/N, T*d]."""
    _, Bl, S, d = recv.shape
    out = np.zeros((Bl, n_tables, d), dtype=recv.dtype)
    for src in range(world):
        for s in range(S):
            t = s * world + src
            if t < n_tables:
                out[:, t, :] = recv[src, :, s, :]
    return out.reshape(Bl, n_tables * d)
