"""The seeded input generator (cvr_synth): determinism and distributions of BASELINE.json's
configs (SURVEY.md §8(d) generator recipe, readings A1-A4, A8).  CPU only."""
import math

import numpy as np
import torch

import cvr_synth as cs


def test_widths():
    assert cs.C1.width == 141 and cs.C2.width == 1728 and cs.C3.width == 12864 and cs.C4.width == 16384


def test_table_rows_counter_based():
    spec = cs.TableSpec(99, 2, 3000, 64, "bf16")
    full = spec.materialize(chunk_rows=1000)
    ids = np.array([2999, 0, 1234, 1234, 77])
    np.testing.assert_array_equal(spec.gather(ids).float().numpy(), full[ids].float().numpy())
    # pure function of (seed, t, row, col): same call twice, different table differs
    assert torch.equal(spec.gather(ids), spec.gather(ids))
    assert not torch.equal(cs.TableSpec(99, 3, 3000, 64, "bf16").gather(ids), spec.gather(ids))


def test_table_rows_distribution():
    x = cs.TableSpec(5, 0, 20000, 64, "f32").materialize().double().numpy().ravel()
    # N(0, 0.01): std 0.1 (A1); 1.28M samples
    assert abs(x.mean()) < 4 * 0.1 / math.sqrt(x.size)
    assert abs(x.std() - 0.1) < 0.002
    # fourth moment of a normal: 3 sigma^4
    assert abs((x ** 4).mean() / x.var() ** 2 - 3.0) < 0.05


def test_zipf_truncated_pmf():
    rng = np.random.default_rng(0)
    n, a, m = 1000, 1.1, 400000
    r = cs.sample_zipf_rows(rng, n, a, m, scramble=False)
    assert r.min() >= 0 and r.max() < n
    H = np.sum(np.arange(1, n + 1, dtype=float) ** -a)
    for k in (1, 2, 10):
        p = k ** -a / H
        f = np.mean(r == k - 1)
        assert abs(f - p) < 5 * math.sqrt(p * (1 - p) / m)


def test_scramble_bijection():
    for n in (1000, 390865, 10_000_000):
        P = cs.scramble_multiplier(n)
        assert math.gcd(P, n) == 1 and P not in (0, 1)
    assert cs.scramble_multiplier(1000) == 761          # SURVEY.md A3 worked value
    k = np.arange(1000)
    assert len(set((k * 761) % 1000)) == 1000


def test_batch_csr_and_lengths():
    bt = cs.make_batch(cs.C2, 3)
    T, B = cs.C2.n_tables, cs.C2.batch
    assert bt.offsets.shape == (T * B + 1,) and bt.offsets[0] == 0 and np.all(np.diff(bt.offsets) >= 1)
    assert bt.nnz == bt.indices.shape[0]
    L = np.diff(bt.offsets)
    assert abs(L.mean() - 4.0) < 0.05                      # Poisson(3)+1
    for t in range(T):
        seg = bt.indices[bt.offsets[t * B]:bt.offsets[(t + 1) * B]]
        assert seg.min() >= 0 and seg.max() < cs.C2.rows[t]
    c1 = cs.make_batch(cs.C1, 0)
    L1 = np.diff(c1.offsets)
    assert L1.min() == 1 and L1.max() == 4
    assert bt.dense.dtype == np.float32 and bt.dense.shape == (B, 64)


def test_batch_deterministic_and_shardable():
    a, b = cs.make_batch(cs.C2, 7, batch=128), cs.make_batch(cs.C2, 7, batch=128)
    np.testing.assert_array_equal(a.indices, b.indices)
    np.testing.assert_array_equal(a.offsets, b.offsets)
    # a table subset (sharded mode) draws the same per-table indices as the full batch
    sub = cs.make_batch(cs.C2, 7, batch=128, tables=[3, 5])
    B = 128
    for j, t in enumerate([3, 5]):
        full_seg = a.indices[a.offsets[t * B]:a.offsets[(t + 1) * B]]
        sub_seg = sub.indices[sub.offsets[j * B]:sub.offsets[(j + 1) * B]]
        np.testing.assert_array_equal(full_seg, sub_seg)


def test_weights_shapes_and_scale():
    w = cs.make_weights(cs.C2)
    assert w["dcn/0/V"].shape == (256, 1728) and w["dcn/0/U"].shape == (1728, 256)
    assert w["mlp/0/W"].shape == (1024, 1728) and w["head/w"].shape == (1, 256)
    assert w["dcn/0/V"].dtype == torch.bfloat16 and w["norm/mean"].dtype == torch.float32
    v = w["dcn/0/V"].double()
    assert abs(v.std().item() - 1 / math.sqrt(1728)) < 0.01 / math.sqrt(1728) * 10
    w1 = cs.make_weights(cs.C1)
    assert w1["dcn/0/W"].shape == (141, 141) and w1["dcn/0/W"].dtype == torch.float32


def test_request_trace():
    t, n = cs.request_trace(2000.0, 2.0)
    assert np.all(np.diff(t) > 0) and t[-1] < 2.0
    assert abs(len(t) - 4000) < 5 * math.sqrt(4000)
    assert n.min() >= 1 and n.max() <= 500
    assert abs(n.mean() - 68.6) < 4.0                      # A21: mean ~ 68.6
