"""Table-wise sharded scoring (BASELINE.json configs[2]).

Tables are placed round-robin (table t on rank t mod N, A18).  Per batch of B_global examples:

  1. every rank pools ITS tables for the GLOBAL batch straight into a destination-major send buffer
     [dst][b_local][t_slot][d] (libcvr ``cvr_embed_shard``; slot = t div N, padded to ceil(T/N)) and
     normalises the dense features of its own batch slice into its local x0;
  2. ``cvr_exchange`` runs the one all-to-all (the only collective on the path) as grouped ncclSend / ncclRecv
     on the library's OWN NCCL communicator (``cvr_comm_init``; the unique id is broadcast by the caller's
     process group, the only thing torch.distributed does here), then
  3. unpacks the received source-major chunks [src][b_local][t_slot][d] into the canonical x0 columns of the
     local slice (V1 of SURVEY.md §8(e));
  4. the dense stage runs data-parallel on the local slice of B_global / N examples.

``FusedShardedScorer`` is V3: step 1 stores pooled rows straight into the owner's x0 over NVLink and steps 2-3
become a per-batch flag handshake.

Pooled values are bit-identical to the unsharded path for every N (the exchange is a copy, P11).
"""
from __future__ import annotations

from typing import Optional, Sequence

import torch
import torch.distributed as dist


def local_tables(n_tables: int, world: int, rank: int):
    return [t for t in range(n_tables) if t % world == rank]


def slots_per_rank(n_tables: int, world: int) -> int:
    return (n_tables + world - 1) // world


def broadcast_unique_id(make, group=None) -> bytes:
    """Rank 0 of ``group`` creates the NCCL unique id (``make()``: libcvr cvr_comm_unique_id) and every rank
    receives it (host plumbing over the caller's process group; gloo in the CPU tests)."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        box = [make() if dist.get_rank(group) == 0 else None]
        dist.broadcast_object_list(box, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
        return box[0]
    return make()


def exchange_handles(blob: bytes, group=None) -> list:
    """Every rank's IPC handle blob (CVR_IPC_HANDLE_BYTES per buffer), in rank order (the host side of V3's peer
    mapping; gloo in the CPU tests, the process group's store-backed object collective on GPUs)."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        out = [None] * dist.get_world_size(group)
        dist.all_gather_object(out, blob, group=group)
        return out
    return [blob]


class FusedShardedScorer:
    """One rank of the V3 sharded path: the gather kernel stores pooled rows
    straight into the owner rank's canonical x0 over NVLink (cvr_embed_fused), per-batch epoch flags replace the
    all-to-all (ready: rows stored; free: the owner's dense stage is done with the slot), and the dense stage waits
    on the ready flags (cvr_wait_peers).  Two x0 slots per rank (epoch parity), so batch e+1's stores overlap
    batch e's dense stage.  No send / receive buffers, no unpack, no NCCL kernel on the data path.

    ``connect(peers=None)``: map the other ranks' slots and flag arrays through CUDA IPC (one process per GPU).
    ``connect(peers=ranks)``: all ranks' FusedShardedScorer objects live in this process (emulated ranks on one
    GPU in the tests)."""

    def __init__(self, cfg, world_size: int, rank: int, batch_global: int, max_nnz: int,
                 device: Optional[torch.device] = None, group=None):
        from ._cvr import CvrModel
        if batch_global % world_size:
            raise ValueError("batch_global must be a multiple of world_size (A18)")
        self.cfg, self.N, self.rank, self.group = cfg, world_size, rank, group
        self.B, self.Bl = batch_global, batch_global // world_size
        self.model = CvrModel(cfg, max_batch=self.Bl, max_nnz=max_nnz, world_size=world_size, rank=rank,
                              device=device)
        self.device = self.model.device
        self.x0 = [self.model.new_x0(self.Bl).zero_() for _ in range(2)]   # slot = epoch % 2
        self.ready = torch.zeros(world_size, dtype=torch.int32, device=self.device)
        self.free = torch.zeros(world_size, dtype=torch.int32, device=self.device)
        self.tables = local_tables(cfg.n_tables, world_size, rank)
        self.epoch = 0
        self.opened = []

    def close(self):
        from ._cvr import ipc_close_handle
        for p in self.opened:
            ipc_close_handle(p)
        self.opened = []

    def _buffers(self):
        return [self.x0[0], self.x0[1], self.ready, self.free]

    def connect(self, peers=None):
        from ._cvr import IPC_HANDLE_BYTES as HB, ipc_get_handle, ipc_open_handle
        if peers is None:
            # each handle carries its tensor's offset inside the caching allocator's block: x0 slots and
            # the 4-int flag arrays are sub-allocated, so the opened base alone would point at the wrong bytes
            mine = [ipc_get_handle(t.data_ptr()) for t in self._buffers()]
            allh = exchange_handles(b"".join(mine), self.group)
            ptrs = []
            for r in range(self.N):
                if r == self.rank:
                    ptrs.append([t.data_ptr() for t in self._buffers()])
                else:
                    ptrs.append([ipc_open_handle(allh[r][HB * i:HB * (i + 1)]) for i in range(4)])
                    self.opened.extend(ptrs[-1])
        else:
            ptrs = [[t.data_ptr() for t in p._buffers()] for p in peers]
        x0_ptrs = [ptrs[r][0] for r in range(self.N)] + [ptrs[r][1] for r in range(self.N)]
        self.model.set_peers(x0_ptrs, [ptrs[r][2] for r in range(self.N)], [ptrs[r][3] for r in range(self.N)],
                             self.ready.data_ptr(), self.free.data_ptr())

    def load_tables(self, tables: Sequence[torch.Tensor]):
        self.model.load_tables(tables, self.tables)

    def load_weights(self, weights):
        self.model.load_weights(weights)

    def embed(self, indices, offsets, dense_local, stream=None):
        """Gather + push this rank's tables for the global batch of the next epoch; signals ready."""
        self.epoch += 1
        self.model.embed_fused(indices, offsets, self.B, dense_local, self.x0[self.epoch % 2], self.epoch,
                               stream=stream)

    def dense(self, scores: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
        """Wait for every rank's rows of this epoch, score the slot, then release it (free flags)."""
        scores = torch.empty(self.Bl, dtype=torch.float32, device=self.device) if scores is None else scores
        self.model.wait_peers(self.epoch, stream=stream)
        self.model.dense(self.x0[self.epoch % 2], self.Bl, scores, stream=stream)
        self.model.release_peers(self.epoch, stream=stream)
        return scores

    def score(self, indices, offsets, dense_local, scores=None, stream=None):
        self.embed(indices, offsets, dense_local, stream)
        return self.dense(scores, stream)


class ShardedScorer:
    """One rank of the sharded scoring path."""

    def __init__(self, cfg, world_size: int, rank: int, batch_global: int, max_nnz: int,
                 device: Optional[torch.device] = None, group=None):
        from ._cvr import CvrModel
        if batch_global % world_size:
            raise ValueError("batch_global must be a multiple of world_size (A18)")
        self.cfg, self.N, self.rank, self.group = cfg, world_size, rank, group
        self.B, self.Bl = batch_global, batch_global // world_size
        self.model = CvrModel(cfg, max_batch=self.Bl, max_nnz=max_nnz, world_size=world_size, rank=rank,
                              device=device)
        self.device = self.model.device
        sb, rb = self.model.shard_buffer_bytes(batch_global)
        # two slots of every per-batch buffer: batch k+1's gather / exchange / unpack overlap batch k's dense stage
        self.send = [torch.empty(sb, dtype=torch.uint8, device=self.device) for _ in range(2)]
        self.recv = [torch.empty(rb, dtype=torch.uint8, device=self.device) for _ in range(2)]
        self.x0 = [self.model.new_x0(self.Bl) for _ in range(2)]
        self.ev_embed = [torch.cuda.Event() for _ in range(2)]
        self.ev_dense = [torch.cuda.Event() for _ in range(2)]
        self.k = 0
        self.tables = local_tables(cfg.n_tables, world_size, rank)
        from ._cvr import comm_unique_id
        self.model.comm_init(broadcast_unique_id(comm_unique_id, group), world_size, rank)

    def load_tables(self, tables: Sequence[torch.Tensor]):
        self.model.load_tables(tables, self.tables)

    def load_weights(self, weights):
        self.model.load_weights(weights)

    def score(self, indices: torch.Tensor, offsets: torch.Tensor, dense_local: torch.Tensor,
              scores: Optional[torch.Tensor] = None, stream=None, s_dense=None) -> torch.Tensor:
        """indices/offsets: this rank's tables over the global batch; dense_local: [B/N, F].

        ``s_dense`` given: the two-stream executor of S9 -- gather, exchange and unpack of this batch on ``stream``
        into buffer slot k % 2 (after the dense stage of batch k-2 released it), the dense stage on ``s_dense``
        after them; back-to-back calls overlap batch k+1's exchange with batch k's dense stage.  ``scores`` must
        stay distinct for the batches in flight.  Without ``s_dense`` everything runs in order on ``stream``."""
        scores = torch.empty(self.Bl, dtype=torch.float32, device=self.device) if scores is None else scores
        s = stream or torch.cuda.current_stream(self.device)
        slot = self.k % 2 if s_dense is not None else 0
        if s_dense is not None and self.k >= 2:
            s.wait_event(self.ev_dense[slot])
        self.model.embed_shard(indices, offsets, self.B, dense_local, self.send[slot], self.x0[slot], stream=s)
        self.model.exchange(self.send[slot], self.recv[slot], self.B, self.x0[slot], stream=s)
        if s_dense is None:
            self.model.dense(self.x0[slot], self.Bl, scores, stream=s)
            return scores
        self.ev_embed[slot].record(s)
        s_dense.wait_event(self.ev_embed[slot])
        self.model.dense(self.x0[slot], self.Bl, scores, stream=s_dense)
        self.ev_dense[slot].record(s_dense)
        self.k += 1
        return scores
