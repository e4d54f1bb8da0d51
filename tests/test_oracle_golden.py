"""Pin the CPU oracle (and the host-side input model) against the reference's outputs.

Golden vectors come from running the real reference (tests/golden/make_golden.py);
the oracle must reproduce them before any GPU result is compared with it.
"""

import hashlib

import numpy as np
import pytest

from conftest import cx, golden_signal
from oracle import ffast as of
from paper_2011_05749_b200.signals import generate_test_case


def test_generate_test_case_bit_identical(golden_ffast):
    for g in golden_ffast["generate_test_case"]:
        x = generate_test_case(g["n"], g["k"], g["snr"], g["seed"]).signal
        digest = hashlib.sha256(np.ascontiguousarray(x, dtype=np.complex128).tobytes()).hexdigest()
        assert digest == g["sha256"], (g["n"], g["k"], g["snr"], g["seed"])


def test_oracle_bucketize_matches_reference(golden_ffast):
    for case in golden_ffast["bucketize"]:
        if "x" in case:
            x = np.array([cx(v) for v in case["x"]])
        else:
            x = golden_signal(case["gen"]).astype(np.complex128)
        got = of.bucket_values(x, case["b"], [case["tau"]])[0]
        want = np.array([cx(v) for v in case["values"]])
        scale = max(1.0, np.max(np.abs(want)))
        assert np.max(np.abs(got - want)) <= 1e-12 * scale


@pytest.mark.parametrize("which", ["small", "c1", "c5"])
def test_oracle_ffast_matches_reference(golden_ffast, which):
    for case in golden_ffast["ffast"]:
        n = case["n"]
        if (which == "c1") != (n == 124950) or (which == "c5") != (n == 2097024):
            continue
        x = golden_signal(case).astype(np.complex128)
        trunc, out = of.ffast(x, case["k"], case["factors"])
        assert abs(of.exact_eps(x) - case["eps"]) <= 1e-12 * case["eps"]
        want = [(f, cx(v)) for f, v in case["recovered"]]
        assert list(out["recovered"].keys()) == [f for f, _ in want]  # same insertion order
        for f, v in want:
            assert abs(out["recovered"][f] - v) <= 1e-12
        assert out["rounds"] == case["rounds"]
        assert out["unresolved"] == case["unresolved"]
        assert list(trunc.keys()) == [f for f, _ in case["truncated"]]


def test_oracle_n20_census_kat():
    # reference tests/test_peeling.py:84-105: 3 zero / 3 single / 3 multi at N=20
    x = generate_test_case(20, 5, "exact", seed=7, positions=[1, 3, 5, 10, 13]).signal
    vals = of.graph_values(x, [4, 5], [0, 1, 2])
    eps = of.exact_eps(x)
    idx = np.array([0, 1, 2, 3, 0, 1, 2, 3, 4])
    b = np.array([4] * 4 + [5] * 5)
    st, f0 = of.classify_rows(vals, idx, b, 20, eps, eps)
    assert list(st) == [of.ZERO, of.MULTI, of.SINGLE, of.SINGLE, of.MULTI, of.SINGLE, of.ZERO,
                        of.MULTI, of.ZERO]
    assert f0[2] == 10 and f0[3] == 3 and f0[5] == 1
