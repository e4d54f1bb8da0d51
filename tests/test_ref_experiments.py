"""The reference's harness tests (pkg/tests/test_bench.py, TestRunCell / TestRunSuite /
TestSublinearityTrend), restated against paper_2011_05749_b200.experiments.  The CLI
and the matplotlib report are out of scope."""

import csv

import numpy as np
import pytest

from paper_2011_05749_b200.experiments import (
    CSV_HEADER,
    ExperimentConfig,
    SkippedCell,
    run_cell,
    run_suite,
)
from paper_2011_05749_b200.peeling import plan_cycles

gpu = pytest.mark.gpu
TIMING = ("runtime_ns", "gbps", "frac_roofline")


def rows_without_timing(path):
    with open(path, newline="") as fh:
        rows = list(csv.DictReader(fh))
    for r in rows:
        for key in TIMING:
            r.pop(key)
    return rows


@gpu
def test_ffast_fixture_cell():
    recs = run_cell("ffast", 20, 5, "exact", trials=3, seed_base=1)
    assert len(recs) == 3 and all(r.success and r.samples_raw == 27 and r.l2 < 1e-9 for r in recs)


@gpu
def test_dense_reads_everything():
    assert all(r.sampled_pct == 1.0 and r.success
               for r in run_cell("dense", 256, 4, "exact", trials=2, seed_base=0))


@gpu
def test_sample_laws():
    for n, k in ((1024, 4), (4096, 8)):
        assert run_cell("dt3", n, k, "exact", 1, 0)[0].samples_raw == (3 * 4 + 12) * 32 * k
    plan, _ = plan_cycles(504, 3, "exact")
    assert run_cell("ffast", 504, 3, "exact", 1, 0)[0].samples_raw == 3 * sum(plan.factors)
    plan, sp = plan_cycles(4095, 4, "noisy", seed=0)
    assert run_cell("rffast", 4095, 4, 20.0, 1, 0)[0].samples_raw == \
        sp.c * sp.m * sum(plan.factors)


def test_incompatible_cells_become_skips():
    skip = run_cell("ffast", 4096, 4, "exact", trials=1, seed_base=0)
    assert isinstance(skip, SkippedCell) and "co-prime" in skip.reason
    skip = run_cell("dt3", 4095, 4, "exact", trials=1, seed_base=0)
    assert isinstance(skip, SkippedCell) and "power-of-two" in skip.reason


@gpu
def test_dt_exact_success_rate_at_large_n():
    assert np.mean([r.success for r in run_cell("dt3", 2 ** 16, 4, "exact", 10, 0)]) >= 0.9


@gpu
def test_suite_csv_header_and_rows(tmp_path):
    out = tmp_path / "suite.csv"
    rows = run_suite(ExperimentConfig(["dt3", "dense"], [256], [2], ["exact"], trials=2,
                                      out_path=str(out)))
    text = out.read_text().splitlines()
    assert text[0] == CSV_HEADER and len(text) == 1 + len(rows) and len(rows) == 4


@gpu
def test_suite_reproducible_modulo_timing(tmp_path):
    def once(p):
        run_suite(ExperimentConfig(["dt2", "ffast"], [256, 504], [3], ["exact", 20.0], trials=2,
                                   seed_base=7, out_path=str(p)))
        return rows_without_timing(p)

    assert once(tmp_path / "a.csv") == once(tmp_path / "b.csv")


def test_skip_row_in_csv(tmp_path):
    out = tmp_path / "s.csv"
    run_suite(ExperimentConfig(["ffast"], [256], [2], ["exact"], out_path=str(out)))
    with open(out, newline="") as fh:
        rows = list(csv.DictReader(fh))
    assert len(rows) == 1 and rows[0]["success"].startswith("skipped(") and rows[0]["seed"] == "-1"


def test_empty_lists_rejected():
    with pytest.raises(ValueError):
        ExperimentConfig(["dt1"], [], [1], ["exact"]).validate()


@gpu
def test_parallel_matches_serial(tmp_path, monkeypatch):
    def once(p):
        run_suite(ExperimentConfig(["dt3", "dsfft"], [256, 512], [2], ["exact"], trials=2,
                                   seed_base=3, out_path=str(p)))
        return rows_without_timing(p)

    monkeypatch.delenv("ALIASFFT_THREADS", raising=False)
    serial = once(tmp_path / "serial.csv")
    monkeypatch.setenv("ALIASFFT_THREADS", "4")
    assert once(tmp_path / "parallel.csv") == serial


@gpu
def test_dt3_unique_samples_nearly_flat_in_n():
    u = {e: np.mean([r.samples_unique for r in run_cell("dt3", 2 ** e, 16, "exact", 3, 0)])
         for e in (12, 14, 16)}
    assert u[16] < 2.5 * u[14] and u[16] < 4 * u[12]
