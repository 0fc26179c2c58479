"""Table-wise sharding host logic on CPU: the sharding simulator reproduces the canonical x0 exactly
for N in {1,2,4,8} (P11), the all-to-all payload is conserved chunk by chunk (P12), and the host plumbing of
the library's NCCL communicator / V3 peer mapping works across a real world_size-2 gloo process group."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import cvr_synth as cs
import oracle as O
from oracle import shard_sim as S


def pooled_c2(B=64):
    cfg = cs.C2
    bt = cs.make_batch(cfg, 3, batch=B)
    return cfg, bt, O.embedding_bag_sum(cs.table_specs(cfg), bt.indices, bt.offsets, cfg.n_tables, B, cfg.dim)


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_simulator_reproduces_canonical_x0(world):
    cfg, bt, pooled = pooled_c2(64)
    sends = [S.build_send(pooled, world, s) for s in range(world)]
    recvs = S.all_to_all(sends)
    Bl = 64 // world
    got = np.concatenate([S.unpack(recvs[d], cfg.n_tables, world) for d in range(world)])
    np.testing.assert_array_equal(got, pooled.reshape(64, -1))


@pytest.mark.parametrize("world", [2, 4, 8])
def test_all_to_all_payload_conserved(world):
    """P12: the all-to-all is a permutation of equal chunks -- the SHA-256 of every (src, dst) chunk sent equals
    the digest of the chunk received, and no byte is created or lost."""
    import hashlib
    cfg, bt, pooled = pooled_c2(64)
    sends = [S.build_send(pooled.astype(np.float32), world, s) for s in range(world)]
    recvs = S.all_to_all(sends)
    dig = lambda a: hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()
    for s_ in range(world):
        for d in range(world):
            assert dig(sends[s_][d]) == dig(recvs[d][s_])
    assert sorted(dig(x[i]) for x in sends for i in range(world)) == sorted(dig(x[i]) for x in recvs
                                                                             for i in range(world))


def test_table_placement_round_robin():
    from paper_2605_29232_b200.sharded import local_tables, slots_per_rank
    assert local_tables(100, 8, 3) == list(range(3, 100, 8))
    assert slots_per_rank(100, 8) == 13 and len(local_tables(100, 8, 7)) == 12
    # every table exactly once across ranks
    assert sorted(t for r in range(8) for t in local_tables(100, 8, r)) == list(range(100))


def test_local_batch_inputs_match_global():
    """Each rank's inputs (its tables over the global batch) are the global batch's per-table draws."""
    from paper_2605_29232_b200.sharded import local_tables
    cfg = cs.C3S.with_(rows=(1000,) * 100)
    full = cs.make_batch(cfg, 0, batch=64)
    for r in range(4):
        loc = cs.make_batch(cfg, 0, batch=64, tables=local_tables(100, 4, r))
        for j, t in enumerate(local_tables(100, 4, r)):
            np.testing.assert_array_equal(loc.indices[loc.offsets[j * 64]:loc.offsets[(j + 1) * 64]],
                                          full.indices[full.offsets[t * 64]:full.offsets[(t + 1) * 64]])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2605_29232_b200.sharded import broadcast_unique_id
    calls = []

    def make():  # stands in for cvr_comm_unique_id (NCCL needs a GPU): only rank 0 may call it
        calls.append(rank)
        return bytes(range(128))

    uid = broadcast_unique_id(make)
    q.put((rank, uid == bytes(range(128)) and calls == ([0] if rank == 0 else [])))
    dist.destroy_process_group()


def test_unique_id_broadcast_gloo_world2():
    """S4 host plumbing: rank 0 alone creates the NCCL unique id for the library's communicator (cvr_comm_init)
    and every rank receives the same 128 bytes over the process group."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert res == {0: True, 1: True}


def _handle_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2605_29232_b200.sharded import exchange_handles
    blob = bytes([rank + 1]) * 288   # stands in for 4 IPC handles (x0 slots 0/1, ready, free: 72 B each)
    got = exchange_handles(blob)
    q.put((rank, got == [bytes([r + 1]) * 288 for r in range(world)]))
    dist.destroy_process_group()


def test_v3_ipc_handle_exchange_gloo_world2():
    """V3 host logic: every rank receives every rank's IPC handle blob in rank order."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_handle_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert res == {0: True, 1: True}
