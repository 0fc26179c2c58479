"""Serving host logic (S0 / S9, config 5): SPEC.md goldens on a simulated clock, nearest-rank
percentiles, and the host batch-assembly entry points of libcvr against a numpy reference."""
import ctypes

import numpy as np
import pytest
import torch

import cvr_synth as cs
from paper_2605_29232_b200.serving import DynamicBatcher, ItemPoolView, Request, nearest_rank, two_stage_schedule


def drive(batcher, arrivals, t_end, dt=1e-4):
    """Simulated clock: submit requests at their arrival times, poll every dt."""
    out, i, t = [], 0, 0.0
    while t <= t_end:
        while i < len(arrivals) and arrivals[i].t_arrival <= t:
            batcher.submit(arrivals[i])
            i += 1
        b = batcher.poll(t)
        if b:
            out.append((round(t, 6), [r.rid for r in b]))
        t += dt
    return out


def test_passthrough_window0_max1():
    reqs = [Request(i, 0.001 * i, 1) for i in range(5)]
    out = drive(DynamicBatcher(max_items=1, window_s=0.0), reqs, 0.01)
    assert [b for _, b in out] == [[0], [1], [2], [3], [4]]


def test_three_requests_one_batch_at_window():
    reqs = [Request(0, 0.0, 1), Request(1, 0.0005, 1), Request(2, 0.0012, 1)]
    out = drive(DynamicBatcher(max_items=8, window_s=0.002), reqs, 0.01)
    assert len(out) == 1 and out[0][1] == [0, 1, 2]
    assert abs(out[0][0] - 0.002) < 2e-4          # dispatched at t0 + timeout


def test_cap_splits_fifo():
    reqs = [Request(0, 0.0, 1), Request(1, 0.0, 1), Request(2, 0.0, 1)]
    out = drive(DynamicBatcher(max_items=2, window_s=0.002), reqs, 0.01)
    assert [b for _, b in out] == [[0, 1], [2]]


def test_whole_requests_never_split_and_fifo():
    rng = np.random.default_rng(0)
    reqs = [Request(i, 0.0001 * i, int(rng.integers(1, 500))) for i in range(300)]
    b = DynamicBatcher(max_items=1000, window_s=0.001)
    out = drive(b, reqs, 1.0)
    flat = [r for _, bb in out for r in bb]
    assert flat == list(range(300))                 # FIFO, each request exactly once
    n = {r.rid: r.n_items for r in reqs}
    for _, bb in out:
        assert sum(n[r] for r in bb) <= 1000


def test_oversized_request_rejected():
    """A request with more items than max_items is rejected at submit (it would overflow the
    server's pinned staging, sized for max_items); the queue keeps serving the others."""
    b = DynamicBatcher(max_items=10, window_s=0.0)
    assert not b.submit(Request(0, 0.0, 11)) and b.rejected == 1
    assert b.submit(Request(1, 0.0, 10))
    assert [r.rid for r in b.poll(0.0)] == [1]


def test_overload_rejects_newest():
    b = DynamicBatcher(max_items=100, window_s=1.0, queue_capacity=2)
    assert b.submit(Request(0, 0, 1)) and b.submit(Request(1, 0, 1))
    assert not b.submit(Request(2, 0, 1)) and b.rejected == 1
    assert [r.rid for r in b.poll(2.0)] == [0, 1]


def test_nearest_rank():
    assert nearest_rank(list(range(1, 101)), 99) == 99
    assert nearest_rank(list(range(1, 101)), 50) == 50
    assert nearest_rank([7.0], 99) == 7.0


def test_two_stage_overlap():   # 2 batches x (5 ms, 5 ms) -> ~15 ms, not 20
    done = two_stage_schedule([5, 5], [5, 5])
    assert done == [10, 15]
    # a single slot serialises A(k) behind B(k-1)
    assert two_stage_schedule([5, 5], [5, 5], slots=1) == [10, 20]


def _ref_gather(pool, ids):
    T, P = pool.n_tables, pool.batch
    off, idx = [0], []
    for t in range(T):
        for i in ids:
            seg = pool.indices[pool.offsets[t * P + i]:pool.offsets[t * P + i + 1]]
            idx.extend(seg)
            off.append(len(idx))
    return np.array(off, np.int32), np.array(idx, np.int32), pool.dense[ids]


def test_gather_items_matches_reference():
    from paper_2605_29232_b200 import build
    build.build()
    cfg = cs.C2
    pool = cs.make_item_pool(cfg, pool_size=512)
    view = ItemPoolView(pool.offsets, pool.indices, pool.dense, cfg.n_tables)
    ids = np.random.default_rng(1).integers(0, 512, 300).astype(np.int32)
    off = torch.empty(cfg.n_tables * 300 + 1, dtype=torch.int32)
    idx = torch.empty(1 << 16, dtype=torch.int32)
    dense = torch.empty(300, cfg.n_dense, dtype=torch.float32)
    nnz = view.gather(ids, off, idx, dense)
    r_off, r_idx, r_dense = _ref_gather(pool, ids)
    assert nnz == len(r_idx)
    np.testing.assert_array_equal(off.numpy(), r_off)
    np.testing.assert_array_equal(idx.numpy()[:nnz], r_idx)
    np.testing.assert_array_equal(dense.numpy(), r_dense)
    with pytest.raises(Exception):
        view.gather(np.array([512], np.int32), off, idx, dense)


def test_concat_requests_matches_reference():
    from paper_2605_29232_b200 import build, lib
    build.build()
    cfg = cs.C1
    reqs = [cs.make_batch(cfg, 40 + i, batch=n) for i, n in enumerate([3, 1, 7])]
    T, F = cfg.n_tables, cfg.n_dense
    B = sum(r.batch for r in reqs)
    n = (ctypes.c_int * 3)(*[r.batch for r in reqs])
    offs = (ctypes.c_void_p * 3)(*[r.offsets.ctypes.data for r in reqs])
    idxs = (ctypes.c_void_p * 3)(*[r.indices.ctypes.data for r in reqs])
    dens = (ctypes.c_void_p * 3)(*[r.dense.ctypes.data for r in reqs])
    o_off = np.zeros(T * B + 1, np.int32)
    o_idx = np.zeros(4096, np.int32)
    o_den = np.zeros((B, F), np.float32)
    nnz = ctypes.c_int64()
    st = lib().cvr_concat_requests(3, T, F, n, offs, idxs, dens, B, o_off.ctypes.data, o_idx.ctypes.data, 4096,
                                   o_den.ctypes.data, ctypes.byref(nnz))
    assert st == 0
    # reference: table-major, requests in order
    r_off, r_idx = [0], []
    for t in range(T):
        for r in reqs:
            for b in range(r.batch):
                seg = r.indices[r.offsets[t * r.batch + b]:r.offsets[t * r.batch + b + 1]]
                r_idx.extend(seg)
                r_off.append(len(r_idx))
    np.testing.assert_array_equal(o_off, r_off)
    np.testing.assert_array_equal(o_idx[:nnz.value], r_idx)
    np.testing.assert_array_equal(o_den, np.concatenate([r.dense for r in reqs]))


def test_request_trace_shapes():
    reqs = cs.make_requests(2000.0, 0.5, 1024)
    assert abs(len(reqs) - 1000) < 5 * 32
    assert all(1 <= len(ids) <= 500 and ids.max() < 1024 for _, ids in reqs)


# ---- Table 6 saturation workload on the simulated clock ------------
def _sim_p99(service, window, max_requests=None, duration=2.0):
    from paper_2605_29232_b200.serving import nearest_rank, simulate_serving

    def at(qps):
        t, n = cs.request_trace(qps, duration, seed=77)
        lat = simulate_serving(t, n, service, 0.0 if window is None else window, max_requests=max_requests)
        return nearest_rank(lat[t >= 0.25 * duration], 99)
    return at


def test_peak_search_bisection_on_step_function():
    from paper_2605_29232_b200.serving import peak_qps_search
    peak, flag = peak_qps_search(lambda q: 0.0 if q <= 1234.0 else 1.0, 0.5, 100.0, 1e5, rel_eps=0.01)
    assert flag == "" and 1234.0 / 1.01 <= peak <= 1234.0
    assert peak_qps_search(lambda q: 1.0, 0.5, 100.0, 1e5) == (0.0, "bound violated at minimal load")


def test_saturation_no_fixed_cost_no_batching_gain():
    """zero per-batch fixed cost -> batching does not amortise anything -> ratio ~ 1."""
    from paper_2605_29232_b200.serving import saturation_table
    svc = lambda n: 4e-6 * n
    rows = saturation_table(lambda w: _sim_p99(svc, w, max_requests=1 if w is None else None), [None, 1e-3],
                            bound_s=10e-3, lo=100.0, hi=20000.0, rel_eps=0.03)
    assert rows[0]["window_ms"] is None and rows[0]["peak_qps"] > 0
    assert 0.8 <= rows[1]["ratio"] <= 1.25, rows


def test_saturation_fixed_cost_batching_raises_peak():
    """delay = F + c n with F >> c -> peak strictly increases with batching (Table 6's shape);
    without batching the server cannot exceed 1 / (F + c E[n]) requests/s."""
    from paper_2605_29232_b200.serving import saturation_table
    F, c = 1e-3, 1e-6
    svc = lambda n: F + c * n
    rows = saturation_table(lambda w: _sim_p99(svc, w, max_requests=1 if w is None else None), [None, 2e-3],
                            bound_s=20e-3, lo=50.0, hi=50000.0, rel_eps=0.03)
    _, n = cs.request_trace(1000.0, 2.0, seed=77)
    assert rows[0]["peak_qps"] <= 1.0 / (F + c * n.mean()) * 1.05
    assert rows[1]["ratio"] > 2.0, rows


# ---- the native batcher (libcvr cvr_batcher_simulate / cvr_serve_trace) pinned to the same contract ---------------
def test_native_batcher_spec_goldens():
    """SPEC.md:639-641 on the native batcher (simulated clock, zero service time)."""
    from paper_2605_29232_b200.serving import batcher_simulate
    # passthrough: window 0, max 1 -> every request its own batch at its arrival
    lat, bof, disp = batcher_simulate([0.000, 0.001, 0.002, 0.003, 0.004], [1] * 5, 0.0, max_items=1)
    assert list(bof) == [0, 1, 2, 3, 4] and np.allclose(disp, [0, 0.001, 0.002, 0.003, 0.004])
    # three requests inside one window -> one batch at t0 + window
    lat, bof, disp = batcher_simulate([0.0, 0.0005, 0.0012], [1, 1, 1], 0.002, max_items=8)
    assert list(bof) == [0, 0, 0] and disp[0] == 0.002
    # cap 2 splits FIFO [2, 1]: the full batch leaves at once, the third at its window
    lat, bof, disp = batcher_simulate([0.0, 0.0, 0.0], [1, 1, 1], 0.002, max_items=2)
    assert list(bof) == [0, 0, 1] and list(disp) == [0.0, 0.002]
    # oversized request and a full queue are rejected (latency +inf, batch -1)
    lat, bof, disp = batcher_simulate([0.0, 0.0, 0.0, 0.0], [11, 1, 1, 1], 0.001, max_items=10, queue_capacity=2)
    assert list(bof) == [-1, 0, 0, -1] and np.isinf(lat[0]) and np.isinf(lat[3])


@pytest.mark.parametrize("window,max_requests", [(0.0, 1), (0.5e-3, 0), (2e-3, 0), (4e-3, 0)])
def test_native_batcher_matches_python_on_traces(window, max_requests):
    """The C++ batcher and serving.DynamicBatcher (via simulate_serving) give the same latency for every request of
    a config-5 trace under a fixed + per-item service model (same rule, same clock arithmetic)."""
    from paper_2605_29232_b200.serving import batcher_simulate, simulate_serving
    t, n = cs.request_trace(20000.0, 0.3, seed=5)
    F, c = 150e-6, 0.02e-6
    ref = simulate_serving(t, n, lambda k: F + c * k, window, max_items=8192,
                           max_requests=max_requests if max_requests else None)
    lat, bof, disp = batcher_simulate(t, n, window, max_items=8192, max_requests=max_requests,
                                      service_fixed_s=F, service_per_item_s=c)
    assert (bof >= 0).all()
    np.testing.assert_array_equal(lat, ref)
