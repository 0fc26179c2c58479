"""bench.py's algorithmic-work formulas (the roofline numerators) against SURVEY.md §8(d)'s per-example table
("Algorithmic work per example": dense FLOP/ex and sparse B/ex, derived there from BASELINE.json's shapes), so the
reported fractions rest on the same work figures the scope table states.  CPU only."""
import os
import sys

import pytest

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import cvr_synth as cs  # noqa: E402


@pytest.mark.parametrize("name,flops", [("c1", 101_732), ("c2", 10_158_592), ("c3s", 67_174_912),
                                        ("c4", 622_855_168)])
def test_dense_flops_per_example_match_survey(name, flops):
    assert bench.dense_flops_per_example(cs.CONFIGS[name]) == flops


def test_c2_sparse_bytes_per_example_match_survey():
    # c2 17,544 B/ex (13,312 of them rows: E[L] = 4 lookups x 26 tables x 128 B) -- an expectation
    # over L ~ Poisson(3) + 1; one seeded batch of 4096 examples lands within 1% of it
    b = cs.make_batch(cs.C2, 0)
    per_ex = bench.embed_bytes(cs.C2, b) / cs.C2.batch
    assert abs(per_ex - 17_544) / 17_544 < 0.01, per_ex


def test_fp32_alu_peak_derivation():
    # 148 SMs x 128 FP32 lanes x 2 FLOP (FFMA) x 1.965 GHz
    assert abs(bench.FP32_ALU_TFLOPS - 74.44992) < 1e-6
