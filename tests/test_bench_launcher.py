"""bench.py's multi-GPU entry on CPU: `--gpus 2` without a torchrun environment
re-launches itself under torch.distributed.run (one process per rank), shards the
signals, all-gathers the result slots and takes the max over ranks — here over gloo
with stand-in slots (--dry-run), since the container has no GPU."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env=None):
    e = dict(os.environ)
    e.pop("WORLD_SIZE", None)
    e.pop("RANK", None)
    e.pop("LOCAL_RANK", None)
    if env:
        e.update(env)
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args,
                       capture_output=True, text=True, timeout=300, env=e, cwd=ROOT)
    return p


def test_gpus2_relaunches_two_ranks_and_gathers():
    p = _run(["--gpus", "2", "--dry-run", "--total-signals", "64", "--steps", "3"])
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout  # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["dry_run"] is True
    assert d["checks"]["gathered_slots_in_rank_order"] is True
    assert d["checks"]["signals_per_rank"] == 32
    assert d["config"]["signals_total"] == 64 and d["config"]["signals_per_rank"] == 32
    assert d["warmup"] >= 3


def test_world_size_mismatch_is_an_error():
    p = _run(["--gpus", "2", "--dry-run"], env={"WORLD_SIZE": "1", "RANK": "0",
                                               "LOCAL_RANK": "0"})
    assert p.returncode == 2 and "WORLD_SIZE" in p.stderr


def test_single_rank_dry_run():
    p = _run(["--dry-run", "--total-signals", "8"])
    assert p.returncode == 0, p.stderr[-3000:]
    d = json.loads([ln for ln in p.stdout.splitlines() if ln.startswith("{")][0])
    assert d["n_gpus"] == 1 and d["checks"]["gathered_slots_in_rank_order"] is True
