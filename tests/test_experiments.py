"""CSV experiment grid (reference bench.py:1-252): schema, skip rows,
case seeds and ledger replay on the host; on the GPU, every row's recovery metrics
equal the oracle's on the same seeded signal."""

import zlib

import numpy as np
import pytest

from paper_2011_05749_b200 import experiments as E


def test_header_keeps_reference_schema_plus_four():
    ref = "algo,n,k,snr,seed,runtime_ns,samples_raw,samples_unique,sampled_pct,l0,l1,l2,success"
    assert E.CSV_HEADER.startswith(ref + ",")
    assert E.CSV_HEADER[len(ref) + 1:].split(",") == ["sectors_bytes", "gbps", "frac_roofline",
                                                      "n_gpus"]


def test_case_seed_is_the_reference_crc32():
    assert E._case_seed(4096, 4, "exact", 0, 1) == zlib.crc32(b"4096|4|exact|0|1")
    assert E._case_seed(4096, 4, 20.0, 3, 0) == zlib.crc32(b"4096|4|20|3|0") ^ 6


def test_config_validation():
    with pytest.raises(ValueError):
        E.ExperimentConfig(["nope"], [8], [1], ["exact"]).validate()
    with pytest.raises(ValueError):
        E.ExperimentConfig(["ffast"], [8], [0], ["exact"]).validate()
    with pytest.raises(ValueError):
        E.ExperimentConfig(["ffast"], [8], [1], ["exact"], trials=0).validate()


def test_skip_rows_run_without_a_gpu(tmp_path):
    # every cell is incompatible (bench.py:114-121): 12 / 24 are not powers of two,
    # 16 / 32 have a single co-prime factor, k = 40 exceeds n
    out = tmp_path / "r.csv"
    rows = E.run_suite(E.ExperimentConfig(["dt2", "dsfft"], [12, 24], [2, 40], ["exact", 10.0],
                                          out_path=str(out)))
    rows += E.run_suite(E.ExperimentConfig(["ffast", "rffast"], [16, 32], [2], ["exact"],
                                           out_path=str(tmp_path / "s.csv")))
    assert all(isinstance(r, E.SkippedCell) for r in rows)
    lines = out.read_text().splitlines()
    assert lines[0] == E.CSV_HEADER and len(lines) == 1 + 2 * 2 * 2 * 2
    assert "dt2,12,2,exact,-1,0,0,0,0,0,0,0,skipped(needs power-of-two n),0,0,0,0" in lines
    assert "dsfft,24,40,10,-1,0,0,0,0,0,0,0,skipped(k exceeds n),0,0,0,0" in lines
    more = (tmp_path / "s.csv").read_text().splitlines()
    assert "ffast,16,2,exact,-1,0,0,0,0,0,0,0,skipped(needs >=2 co-prime factors of n),0,0,0,0" \
        in more


@pytest.mark.gpu
def test_grid_rows_match_the_oracle(tmp_path):
    from oracle import dsfft as od
    from oracle import ffast as of
    from oracle import oneshot as oo
    from paper_2011_05749_b200 import OneShotConfig, SparseSpectrum, evaluate, generate_test_case
    from paper_2011_05749_b200.peeling import plan_cycles

    cfg = E.ExperimentConfig(["dt2", "dsfft", "dense"], [4096], [4], ["exact"],
                             trials=2, out_path=str(tmp_path / "g.csv"))
    rows = E.run_suite(cfg)
    rows += E.run_suite(E.ExperimentConfig(["ffast"], [4095], [4], ["exact"], trials=2,
                                           out_path=str(tmp_path / "f.csv")))
    assert all(isinstance(r, E.ExperimentRecord) for r in rows)
    for r in rows:
        case = generate_test_case(r.n, r.k, r.snr, r.seed)
        x = case.signal
        if r.algo == "ffast":
            plan, _ = plan_cycles(r.n, r.k, "exact")
            est, _ = of.ffast(x, r.k, plan.factors)
        elif r.algo == "dt2":
            c = OneShotConfig.default(r.n, r.k, variant="dt2", seed=r.seed)
            est, _, _ = oo.sfft_dt(x, r.k, c.b, c.a_m, c.p, "dt2", r.seed)
        elif r.algo == "dsfft":
            est, _, _ = od.dsfft(x, r.k, "exact", r.seed)
        else:
            spec = np.fft.fft(x) / r.n
            order = np.argsort(-np.abs(spec), kind="stable")[: r.k]
            est = {int(f): complex(spec[f]) for f in order}
        m = evaluate(case.truth, SparseSpectrum(r.n, est))
        assert (r.l0, r.success) == (m.l0, m.l0 == 0), r
        assert abs(r.l1 - m.l1) <= 1e-6 * max(1.0, m.l1) and abs(r.l2 - m.l2) <= 1e-6 * max(1.0, m.l2)
        assert r.samples_raw > 0 and 0 < r.samples_unique <= r.n
        assert r.sectors_bytes >= 32 and r.gbps > 0 and r.n_gpus == 1
    text = (tmp_path / "g.csv").read_text().splitlines()
    assert len(text) == 1 + 3 * 2
