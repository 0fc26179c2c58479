"""Serving machinery of the scoring path (config 5):

* ``DynamicBatcher`` -- server-side dynamic batching with a coalescing window (PAPER.md:1560
  "Server-Side Batching dynamically aggregates independent requests", Table 6).
  Requests (one query's candidate items each: "Client-Side Batching") are queued FIFO and dispatched
  as the longest FIFO prefix of WHOLE requests with at most ``max_items`` items, either when the queue
  holds >= max_items items or when the oldest queued request has waited ``window_s`` (window anchored
  at the oldest request; requests never split or reordered).  A full queue rejects the
  newest request (CVR_E_OVERLOAD semantics).
* ``nearest_rank`` -- percentile by nearest rank.
* ``two_stage_schedule`` -- the simulated-clock model of the decoupled two-stage executor (S9):
  stage A of batch k+1 overlaps stage B of batch k, with ``slots`` x0 buffers.
* ``Server`` -- the real loop, native (libcvr ``cvr_serve_trace``): admits requests at their scheduled (open-loop)
  arrival times into the same batcher (C++), assembles each batch on the host (``cvr_gather_items`` into pinned
  staging, stage 0), scores it through ``cvr_score_host`` (H2D -> embed stream -> dense stream -> zero-copy
  scores, S1-S8) and stamps completion when the batch's event has fired.  Latency = completion - scheduled arrival.
  ``batcher_simulate`` replays the native batcher on a simulated clock (tests pin it to DynamicBatcher).
* ``simulate_serving`` / ``peak_qps_search`` / ``saturation_table`` -- the Table 6 workload (
  SPEC.md:660-668): for each coalescing window, the highest offered load whose p99
  latency stays under a bound (bisection), and its ratio to the no-batching row.

Host logic only: every score is computed by libcvr's kernels.
"""
from __future__ import annotations

import collections
import ctypes
import math
import time
from dataclasses import dataclass
from typing import Deque, List, Optional, Sequence

import numpy as np
import torch

from ._cvr import CvrError, lib

CVR_E_OVERLOAD = 9


@dataclass
class Request:
    rid: int
    t_arrival: float          # scheduled arrival time (s, open loop)
    n_items: int
    item_ids: Optional[np.ndarray] = None   # pool item ids (serving benchmark)


class DynamicBatcher:
    def __init__(self, max_items: int = 8192, window_s: float = 0.002, queue_capacity: int = 1 << 16,
                 max_requests: Optional[int] = None):
        """``max_requests = 1`` with ``window_s = 0`` is Table 6's "0ms (w/o dynamic batching)" row: every
        request is its own batch, dispatched as soon as the server can take it."""
        if max_items < 1 or window_s < 0 or queue_capacity < 1 or (max_requests is not None and max_requests < 1):
            raise ValueError("max_items >= 1, window_s >= 0, queue_capacity >= 1, max_requests >= 1")
        self.max_items, self.window_s, self.capacity = max_items, window_s, queue_capacity
        self.max_requests = max_requests
        self.q: Deque[Request] = collections.deque()
        self.items = 0
        self.rejected = 0

    def __len__(self):
        return len(self.q)

    def submit(self, req: Request) -> bool:
        """Queue a request; False if the queue is full (overload) or the request alone holds more
        than max_items items (requests are never split, so it could never be dispatched within the batch cap that
        the server's staging and the library's max_batch are sized for)."""
        if len(self.q) >= self.capacity or req.n_items > self.max_items:
            self.rejected += 1
            return False
        self.q.append(req)
        self.items += req.n_items
        return True

    def next_deadline(self) -> Optional[float]:
        return self.q[0].t_arrival + self.window_s if self.q else None

    def poll(self, now: float) -> Optional[List[Request]]:
        """The batch to dispatch at time ``now``, or None."""
        if not self.q:
            return None
        if self.items < self.max_items and now < self.q[0].t_arrival + self.window_s:
            return None
        out, n = [], 0
        while self.q and n + self.q[0].n_items <= self.max_items and \
                (self.max_requests is None or len(out) < self.max_requests):
            r = self.q.popleft()
            n += r.n_items
            out.append(r)
        self.items -= n
        return out


def nearest_rank(samples: Sequence[float], p: float) -> float:
    """Nearest-rank percentile: the ceil(p/100 * N)-th smallest sample (1-based)."""
    s = sorted(samples)
    if not s:
        return float("nan")
    k = max(1, math.ceil(p / 100.0 * len(s)))
    return s[k - 1]


def two_stage_schedule(a_costs: Sequence[float], b_costs: Sequence[float], slots: int = 2, t0: float = 0.0):
    """Completion times of batches through a two-stage pipeline (stage A on one resource, stage B on
    another): A(k) starts when A(k-1) is done and its x0 slot is free (B(k-slots) done); B(k) starts
    when A(k) and B(k-1) are done."""
    a_done, b_done = [], []
    for k, (a, b) in enumerate(zip(a_costs, b_costs)):
        start_a = max(t0, a_done[-1] if a_done else t0, b_done[k - slots] if k >= slots else t0)
        a_done.append(start_a + a)
        start_b = max(a_done[-1], b_done[-1] if b_done else t0)
        b_done.append(start_b + b)
    return b_done


def simulate_serving(arrivals: Sequence[float], n_items: Sequence[int], service, window_s: float,
                     max_items: int = 8192, max_requests: Optional[int] = None) -> np.ndarray:
    """Simulated-clock serving: DynamicBatcher in front of ONE server whose batch of n items
    takes ``service(n)`` seconds; a batch is dispatched when the batcher releases it and the server is free.
    Returns per-request latency (completion - arrival)."""
    b = DynamicBatcher(max_items, window_s, queue_capacity=1 << 30, max_requests=max_requests)
    lat = np.zeros(len(arrivals))
    i, now, free_at, N = 0, 0.0, 0.0, len(arrivals)
    done = 0
    while done < N:
        # next event: an arrival, the oldest request's window expiring, or the server freeing up
        cands = []
        if i < N:
            cands.append(arrivals[i])
        if len(b):
            cands.append(max(b.next_deadline(), free_at) if b.items < max_items else free_at)
        now = max(now, min(cands))
        while i < N and arrivals[i] <= now:
            b.submit(Request(i, arrivals[i], int(n_items[i])))
            i += 1
        if now >= free_at:
            batch = b.poll(now)
            if batch:
                n = sum(r.n_items for r in batch)
                free_at = now + service(n)
                for r in batch:
                    lat[r.rid] = free_at - r.t_arrival
                done += len(batch)
                continue
        if i >= N and len(b) and now < free_at:
            now = free_at
    return lat


def peak_qps_search(p99_at, bound_s: float, lo: float, hi: float, rel_eps: float = 0.05, max_iter: int = 30,
                    confirm: int = 0):
    """the highest offered load whose measured p99 <= bound, by bisection (geometric, until
    hi/lo <= 1 + rel_eps).  ``p99_at(qps) -> seconds``.  Returns (peak, flag): peak 0.0 and flag 'bound
    violated at minimal load' if even ``lo`` violates the bound; flag 'hi feasible' if the whole range is.
    ``confirm``: re-measure the result up to that many times, stepping down by (1 + rel_eps) on a violation
    (measured p99 is noisy, and with long windows it is not monotone in the load: a full batch dispatches
    before its window expires)."""
    lo0 = lo
    if p99_at(lo) > bound_s:
        return 0.0, "bound violated at minimal load"
    if p99_at(hi) <= bound_s:
        return hi, "hi feasible"
    for _ in range(max_iter):
        if hi / lo <= 1.0 + rel_eps:
            break
        mid = math.sqrt(lo * hi)
        if p99_at(mid) <= bound_s:
            lo = mid
        else:
            hi = mid
    for _ in range(confirm):
        if lo <= lo0 or p99_at(lo) <= bound_s:
            break
        lo = max(lo0, lo / (1.0 + rel_eps))
    return lo, ""


def saturation_table(p99_for_window, windows_s: Sequence[Optional[float]], bound_s: float, lo: float, hi: float,
                     rel_eps: float = 0.05, confirm: int = 0):
    """Table 6 layout: one row per window (None = no dynamic batching, the first row);
    ``p99_for_window(window) -> (qps -> p99 seconds)``; ratio = peak / the no-batching row's peak."""
    rows = []
    for w in windows_s:
        peak, flag = peak_qps_search(p99_for_window(w), bound_s, lo, hi, rel_eps, confirm=confirm)
        rows.append({"window_ms": None if w is None else w * 1e3, "peak_qps": peak, "flag": flag})
    base = rows[0]["peak_qps"] if rows else 0.0
    for r in rows:
        r["ratio"] = r["peak_qps"] / base if base > 0 else None
    return rows


class ItemPoolView:
    """A host-resident item pool in the library's CSR layout (table-major offsets [T*P+1])."""

    def __init__(self, offsets: np.ndarray, indices: np.ndarray, dense: np.ndarray, n_tables: int):
        self.P = dense.shape[0]
        self.T, self.F = n_tables, dense.shape[1]
        self.offsets = np.ascontiguousarray(offsets, dtype=np.int32)
        self.indices = np.ascontiguousarray(indices, dtype=np.int32)
        self.dense = np.ascontiguousarray(dense, dtype=np.float32)
        assert self.offsets.shape == (self.T * self.P + 1,)

    def gather(self, item_ids: np.ndarray, out_off: torch.Tensor, out_idx: torch.Tensor, out_dense: torch.Tensor) -> int:
        """Assemble the batch (cvr_gather_items) into the given (pinned) host tensors; returns nnz."""
        ids = np.ascontiguousarray(item_ids, dtype=np.int32)
        nnz = ctypes.c_int64()
        st = lib().cvr_gather_items(self.T, self.F, self.P, self.offsets.ctypes.data, self.indices.ctypes.data,
                                    self.dense.ctypes.data, len(ids), ids.ctypes.data, out_dense.shape[0],
                                    out_off.data_ptr(), out_idx.data_ptr(), out_idx.numel(), out_dense.data_ptr(),
                                    ctypes.byref(nnz))
        if st:
            raise CvrError(st, "cvr_gather_items")
        return nnz.value


def batcher_simulate(t_arrival, n_items, window_s: float, max_items: int = 8192, max_requests: int = 0,
                     queue_capacity: int = 1 << 30, service_fixed_s: float = 0.0, service_per_item_s: float = 0.0):
    """libcvr cvr_batcher_simulate: the native batcher on a simulated clock -> (latency, batch_of, dispatch_times)."""
    t = np.ascontiguousarray(t_arrival, dtype=np.float64)
    n = np.ascontiguousarray(n_items, dtype=np.int32)
    N = len(t)
    lat, bof, disp = np.zeros(N), np.zeros(N, np.int32), np.zeros(max(N, 1))
    nb = ctypes.c_int()
    st = lib().cvr_batcher_simulate(N, t.ctypes.data, n.ctypes.data, window_s, max_items, max_requests or 0,
                                    queue_capacity, service_fixed_s, service_per_item_s, lat.ctypes.data,
                                    bof.ctypes.data, disp.ctypes.data, ctypes.byref(nb))
    if st:
        raise CvrError(st, "cvr_batcher_simulate")
    return lat, bof, disp[:nb.value]


class Server:
    """Open-loop serving of a request trace: libcvr's native loop (cvr_serve_trace: the batcher above in C++,
    host batch assembly into page-locked slots, cvr_score_host on three streams, completion by CUDA events, one
    busy-polling host thread).  This class only marshals the trace and the results."""

    def __init__(self, model, pool: ItemPoolView, max_items: int = 8192, window_s: float = 0.002,
                 host_slots: int = 3, max_nnz: Optional[int] = None, max_requests: Optional[int] = None,
                 use_graphs: bool = True, queue_capacity: int = 1 << 16):
        self.m, self.pool = model, pool
        # The executor replays one CUDA graph per stage and x0 slot for every batch (the batch's pointers and size
        # live in a device-side call block), so dynamically sized batches need no capture after the first two.
        model.set_option("graphs", 1 if use_graphs else 0)
        if max_items > model.max_batch:
            raise ValueError(f"max_items {max_items} > the model's max_batch {model.max_batch}")
        from ._cvr import cvr_serve_config
        self.cfg = cvr_serve_config(window_s, max_items, max_requests or 0, queue_capacity, host_slots,
                                    max_nnz or model.max_nnz, 0.0)
        self.max_items = max_items
        self.batcher = type("BatcherStats", (), {"rejected": 0})()
        dev = model.device
        self.s_copy, self.s_embed = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        self.s_dense = torch.cuda.Stream(dev, priority=-1)
        self.stats = None
        if use_graphs:  # capture every grid-size bucket's graphs now: no batch of a run pays a capture
            model.warm_graphs(max_items, self.s_embed, self.s_dense)

    def run(self, reqs: List[Request], keep_scores: bool = False, abort_after_s: Optional[float] = None):
        """Serve the trace; returns (latency [s] per request id, batch sizes, {rid: scores} or None).
        ``abort_after_s``: stop early (remaining requests get latency +inf) once the oldest queued request has
        waited that long -- an overloaded point of a saturation search."""
        reqs = sorted(reqs, key=lambda r: r.rid)
        N = len(reqs)
        t = np.array([r.t_arrival for r in reqs], np.float64)
        n = np.array([r.n_items for r in reqs], np.int32)
        start = np.zeros(N + 1, np.int64)
        start[1:] = np.cumsum(n)
        ids = np.concatenate([np.asarray(r.item_ids, np.int32) for r in reqs]) if N else np.zeros(1, np.int32)
        lat, sizes, scores = self.run_arrays(t, n, start, ids, keep_scores, abort_after_s)
        out = None
        if keep_scores:
            out = {r.rid: scores[start[i]:start[i + 1]].copy() for i, r in enumerate(reqs)}
        return lat, sizes, out

    def run_arrays(self, t, n, start, ids, keep_scores: bool = False, abort_after_s: Optional[float] = None):
        """The trace as flat arrays (t_arrival, n_items, item_start [N+1], item_ids): (latency, batch sizes,
        scores [sum n] or None)."""
        from ._cvr import cvr_serve_stats
        t = np.ascontiguousarray(t, np.float64)
        n = np.ascontiguousarray(n, np.int32)
        start = np.ascontiguousarray(start, np.int64)
        ids = np.ascontiguousarray(ids, np.int32) if len(ids) else np.zeros(1, np.int32)
        N = len(t)
        lat = np.zeros(N)
        sizes = np.zeros(max(N, 1), np.int32)
        scores = np.zeros(max(int(start[-1]), 1), np.float32) if keep_scores else None
        nb = ctypes.c_int()
        stats = cvr_serve_stats()
        self.cfg.abort_after_s = abort_after_s or 0.0
        torch.cuda.synchronize()
        p = self.pool
        st = lib().cvr_serve_trace(self.m.h, ctypes.byref(self.cfg), p.T, p.F, p.P, p.offsets.ctypes.data,
                                   p.indices.ctypes.data, p.dense.ctypes.data, N, t.ctypes.data, n.ctypes.data,
                                   start.ctypes.data, ids.ctypes.data, lat.ctypes.data,
                                   scores.ctypes.data if keep_scores else None, sizes.ctypes.data, ctypes.byref(nb),
                                   ctypes.byref(stats), self.s_copy.cuda_stream, self.s_embed.cuda_stream,
                                   self.s_dense.cuda_stream)
        if st:
            self.m._check(st)
        self.batcher.rejected = stats.rejected
        self.stats = {"rejected": stats.rejected, "aborted": bool(stats.aborted), "items_served": stats.items_served,
                      "host_dispatch_s": stats.host_dispatch_s, "wall_s": stats.wall_s,
                      "max_dispatch_s": stats.max_dispatch_s, "max_gather_s": stats.max_gather_s, "loop_gaps_1ms": stats.loop_gaps_1ms}
        return lat, sizes[:nb.value], scores
