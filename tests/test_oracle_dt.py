"""Pin the sFFT-DT oracle against reference goldens (CPU only).

Parity definition: vote counts identical; the significant support
{|v| > 1e-3} identical with values within 1e-9; zero-magnitude padding entries
(the reference's own ulp-chaotic filler) are not compared.
"""

import numpy as np
import pytest

from conftest import cx, dt_signal
from oracle import oneshot as od

SIG = 1e-3


def significant(pairs):
    return {f: cx(v) for f, v in pairs if abs(cx(v)) > SIG}


@pytest.mark.parametrize("idx", range(19))
def test_oracle_sfft_dt(golden_dt, idx):
    case = golden_dt["cases"][idx]
    x = dt_signal(case).astype(np.complex128)
    trunc, entries, counts = od.sfft_dt(x, case["k"], case["b"], 4, case["p"], case["variant"],
                                        case["seed"])
    assert [[int(i), int(counts[i])] for i in np.flatnonzero(counts)] == case["counts_nz"]
    want = significant(case["entries"])
    got = {f: v for f, v in entries.items() if abs(v) > SIG}
    assert set(got) == set(want)
    for f, v in want.items():
        assert abs(got[f] - v) <= 1e-9
    assert {f for f, v in trunc.items() if abs(v) > SIG} == set(significant(case["truncated"]))
