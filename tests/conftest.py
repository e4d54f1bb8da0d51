"""Test configuration: the `gpu` marker, golden fixtures, seeded inputs.

`-m "not gpu"` tests run on any host (oracle vs goldens, host logic, ABI
exports); `-m gpu` tests call the CUDA library and are skipped, not failed, when
no CUDA device is visible.
"""

import json
import os
import sys
import zlib

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device")
    try:
        from hypothesis import settings

        settings.register_profile("deterministic", derandomize=True, deadline=None)
        settings.load_profile("deterministic")
    except ImportError:  # pragma: no cover
        pass


def pytest_collection_modifyitems(config, items):
    import torch

    if torch.cuda.is_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device visible")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


def load_golden(name: str) -> dict:
    with open(os.path.join(GOLDEN_DIR, name)) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def golden_ffast():
    return load_golden("golden_ffast.json")


def cx(pair) -> complex:
    return complex(pair[0], pair[1])


def case_seed(n, k, snr, seed_base, trial):
    """The reference bench seed convention (bench.py:123-127)."""
    tag = "exact" if snr == "exact" else f"{float(snr):.9g}"
    return zlib.crc32(f"{n}|{k}|{tag}|{seed_base}|{trial}".encode()) ^ (seed_base << 1)


def golden_signal(gen: dict) -> np.ndarray:
    """Regenerate a golden case's input with the package's (pinned) input model."""
    from paper_2011_05749_b200.signals import generate_test_case

    x = generate_test_case(gen["n"], gen["k"], gen["snr"], gen["seed"],
                           positions=gen.get("positions")).signal
    if gen.get("c64"):
        x = x.astype(np.complex64)
    return x


@pytest.fixture
def rng():
    return np.random.default_rng(12345)


@pytest.fixture(scope="session")
def golden_rffast():
    return load_golden("golden_rffast.json")


def search_plan_of(case):
    """SearchPlan of a golden R-FFAST run (anchors as captured from the reference)."""
    from paper_2011_05749_b200.peeling import SearchPlan, kay_weights

    return SearchPlan(c=case["c"], m=case["m"], anchors=list(case["anchors"]),
                      weights=kay_weights(case["m"]))


@pytest.fixture(scope="session")
def golden_dt():
    return load_golden("golden_dt.json")


def dt_signal(case):
    from paper_2011_05749_b200.signals import generate_test_case

    x = generate_test_case(case["n"], case["k"], case["snr"], case["seed"]).signal
    return x.astype(np.complex64) if case.get("c64") else x


@pytest.fixture(scope="session")
def golden_dsfft():
    return load_golden("golden_dsfft.json")


def dsfft_signal(case):
    from paper_2011_05749_b200.signals import generate_test_case

    x = generate_test_case(case["n"], case["k"], case["snr"], case["seed"],
                           positions=case.get("positions")).signal
    return x.astype(np.complex64) if case.get("c64") else x


# ---- fixtures mirroring the reference suite's inputs (tests/conftest.py of the
# reference: the same seeds and fixed tone positions, regenerated with our model)

@pytest.fixture
def five_tone_n20():
    """20-point exact case with tones at {1, 3, 5, 10, 13}."""
    from paper_2011_05749_b200 import generate_test_case

    return generate_test_case(20, 5, "exact", seed=7, positions=[1, 3, 5, 10, 13])


@pytest.fixture
def five_tone_n64():
    """64-point exact case with tones at {1, 6, 13, 20, 59}."""
    from paper_2011_05749_b200 import generate_test_case

    return generate_test_case(64, 5, "exact", seed=11, positions=[1, 6, 13, 20, 59])


def brute_dft(x):
    """O(n^2) forward transform, 1/n scaled (independent of every FFT under test)."""
    x = np.asarray(x, dtype=np.complex128)
    n = x.size
    idx = np.arange(n)
    return np.exp(-2j * np.pi * np.outer(idx, idx) / n) @ x / n


def alias_sum(spectrum, b, tau):
    """Bucket values from a full spectrum: sum over the residue class of i mod b of
    X[f] * w^(tau f) (the aliasing identity, evaluated term by term)."""
    spectrum = np.asarray(spectrum, dtype=np.complex128)
    n = spectrum.size
    out = np.zeros(b, dtype=np.complex128)
    for f in range(n):
        out[f % b] += spectrum[f] * np.exp(-2j * np.pi * ((tau * f) % n) / n)
    return out
