"""Pin the R-FFAST oracle against reference goldens (CPU only)."""

import numpy as np
import pytest

from conftest import cx, search_plan_of
from oracle import ffast as of
from oracle import rffast as orf
from paper_2011_05749_b200.signals import generate_test_case


def test_oracle_singleton_search(golden_rffast):
    for s in golden_rffast["searches"]:
        sp = search_plan_of(s)
        y = np.array([cx(v) for v in s["residual"]])
        f0, v, rn = orf.search(y, s["index"], s["b"], s["n"], sp.c, sp.m, sp.weights, sp.shifts)
        assert f0 == s["f0"]
        assert abs(v - cx(s["value"])) <= 1e-12
        assert abs(rn - s["resnorm"]) <= 1e-12 * max(1.0, s["resnorm"])


@pytest.mark.parametrize("idx", range(7))
def test_oracle_noisy_runs(golden_rffast, idx):
    case = golden_rffast["runs"][idx]
    sp = search_plan_of(case)
    x = generate_test_case(case["n"], case["k"], case["snr"], case["seed"]).signal
    vals = of.graph_values(x, case["factors"], sp.shifts)
    t0, t1 = orf.thresholds(orf.node_energies(vals), len(sp.shifts))
    assert (t0, t1) == (case["t0"], case["t1"])
    out = orf.peel_noisy(vals, case["factors"], case["n"], sp.c, sp.m, sp.weights, sp.shifts, t0,
                         t1, case["k"] + 4)
    assert list(out["recovered"]) == [f for f, _ in case["recovered"]]
    for f, v in case["recovered"]:
        assert abs(out["recovered"][f] - cx(v)) <= 1e-12
    assert out["rounds"] == case["rounds"] and out["unresolved"] == case["unresolved"]
