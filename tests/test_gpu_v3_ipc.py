"""V3 across two real processes: the fused exchange's peer mapping goes through CUDA IPC
(cvr_ipc_get_handle / cvr_ipc_open_handle, handles carrying each tensor's offset inside its caching-allocator
block), the gather kernel of each process stores pooled rows straight into the OTHER process's x0 slot, and the
ready / free epoch flags are written across processes with system-scope release / acquire.

Both processes share the one GPU of this box.  Their launches are sequenced by host barriers so that no kernel
ever waits on a flag that a later launch will set (every spin-wait finds its flag already published): rank 0's
gather, then rank 1's gather, then both dense stages.  Four epochs cover both x0 slots and the free-slot handshake
(epochs 3 and 4 wait on the free flags released by epochs 1 and 2).  Each rank's x0 slice and scores must be
bit-identical to the unsharded path (P11)."""
import os
import socket

import pytest
import torch

pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import numpy as np  # noqa: F401
    import torch.distributed as dist

    import cvr_synth as cs
    from paper_2605_29232_b200 import CvrModel
    from paper_2605_29232_b200.sharded import FusedShardedScorer, local_tables
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        cfg = cs.C3.with_(rows=(20000,) * 100)
        B, Bl = 256, 256 // world
        tabs = [s.materialize(device="cuda") for s in cs.table_specs(cfg)]
        w = cs.make_weights(cfg)
        ref = CvrModel(cfg, max_batch=B, max_nnz=1 << 20)
        ref.load_tables(tabs)
        ref.load_weights({k: v.cuda() for k, v in w.items()})
        sc = FusedShardedScorer(cfg, world, rank, B, 1 << 20)
        sc.connect()  # real CUDA IPC: handles exchanged over the gloo group, opened in this process
        assert len(sc.opened) == 4 * (world - 1)
        sc.load_tables([tabs[t] for t in sc.tables])
        sc.load_weights({k: v.cuda() for k, v in w.items()})
        torch.cuda.synchronize()
        msgs = []
        for epoch in (1, 2, 3, 4):
            bt = cs.make_batch(cfg, 40 + epoch, batch=B)
            idx, off, dense = (torch.from_numpy(bt.indices).cuda(), torch.from_numpy(bt.offsets).cuda(),
                               torch.from_numpy(bt.dense).cuda())
            x0_ref = ref.embed(idx, off, B, dense)
            s_ref = ref.dense(x0_ref, B)
            lb = cs.make_batch(cfg, 40 + epoch, batch=B, tables=local_tables(cfg.n_tables, world, rank))
            li, lo = torch.from_numpy(lb.indices).cuda(), torch.from_numpy(lb.offsets).cuda()
            dl = dense[rank * Bl:(rank + 1) * Bl].contiguous()
            torch.cuda.synchronize()
            for r in range(world):  # gathers in rank order: each one's free-flag wait is already satisfied
                dist.barrier()
                if r == rank:
                    sc.embed(li, lo, dl)
                    torch.cuda.synchronize()
            dist.barrier()  # every rank's rows (and ready flags) have landed in every owner's slot
            s = sc.dense()
            torch.cuda.synchronize()
            dist.barrier()  # every dense stage done (free flags released) before the next epoch's gathers
            if sc.model.status() != 0:
                msgs.append(f"epoch {epoch}: CVR_E_INDEX")
            if int(sc.ready.min()) != epoch or int(sc.free.min()) != epoch:
                msgs.append(f"epoch {epoch}: flags ready={sc.ready.tolist()} free={sc.free.tolist()}")
            if not torch.equal(sc.x0[epoch % 2], x0_ref[rank * Bl:(rank + 1) * Bl]):
                msgs.append(f"epoch {epoch}: x0 differs")
            if not torch.equal(s, s_ref[rank * Bl:(rank + 1) * Bl]):
                msgs.append(f"epoch {epoch}: scores differ")
        sc.close()
        dist.destroy_process_group()
        q.put((rank, msgs))
    except Exception as e:  # noqa: BLE001
        q.put((rank, [f"exception: {e!r}"]))


def test_v3_two_processes_ipc_bitexact():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=600) for _ in ps)
    for p in ps:
        p.join(timeout=120)
    assert res == {0: [], 1: []}, res
