"""Pin the DSFFT oracle against reference goldens (CPU only): layer trace, output
support and values, plus the reference's layer-count KAT."""

import numpy as np
import pytest

from conftest import cx, dsfft_signal
from oracle import dsfft as odf


@pytest.mark.parametrize("idx", range(13))
def test_oracle_dsfft(golden_dsfft, idx):
    case = golden_dsfft["cases"][idx]
    x = dsfft_signal(case).astype(np.complex128)
    trunc, _, trace = odf.dsfft(x, case["k"], case["mode"], case["seed"], case["noise_std"])
    assert trace == case["trace"]
    want = {f: cx(v) for f, v in case["truncated"]}
    assert set(trunc) == set(want)
    for f, v in want.items():
        assert abs(trunc[f] - v) <= 1e-9


def test_layer_count_kat(golden_dsfft):
    from paper_2011_05749_b200 import generate_test_case

    x = generate_test_case(64, 5, "exact", seed=11, positions=[1, 6, 13, 20, 59]).signal
    layer = odf.initial(x, 0, 1e-6)
    counts = [len(layer[2])]
    for _ in range(3):
        layer = odf.expand(x, layer, 1e-6)
        counts.append(len(layer[2]))
    assert counts == golden_dsfft["layer_counts_n64"] == [1, 2, 4, 5]
