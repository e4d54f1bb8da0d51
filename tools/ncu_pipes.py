#!/usr/bin/env python
"""FP64 work and pipe use of the compute-bound configs, counted by ncu.

    python tools/ncu_pipes.py [--configs c2,c3,c3auto,c4dt3,c4dsfft] [--out profiles/r02_pipes.json]

For each config, a child process synthesises the bench's inputs (bench.synth_batch),
runs the batched call once to warm up, then once more between cudaProfilerStart /
Stop; ncu (--profile-from-start off, --clock-control none) records every kernel of
that one call with

  gpu__time_duration.sum                                  kernel time
  sm__sass_thread_inst_executed_op_{dadd,dmul,dfma}_pred_on.sum   FP64 thread ops
  sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active    FP64 pipe busy
  sm__inst_issued.avg.pct_of_peak_sustained_active                issue slots used

and the parent writes, per config: FP64 flops per signal (dadd + dmul + 2 dfma,
summed over the call's kernels — the numerator bench.py divides by its live
CUDA-event time), and per kernel its time share, FP64 pipe % and issue %.  ncu's
per-kernel times are serialised and cold-cache: only the shares are used.
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

METRICS = [
    "gpu__time_duration.sum",
    "sm__sass_thread_inst_executed_op_dadd_pred_on.sum",
    "sm__sass_thread_inst_executed_op_dmul_pred_on.sum",
    "sm__sass_thread_inst_executed_op_dfma_pred_on.sum",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_issued.avg.pct_of_peak_sustained_active",
]
SIGNALS = {"c2": 64, "c3": 16, "c3auto": 16, "c4dt3": 32, "c4dsfft": 8}


def child(name):
    import numpy as np
    import torch

    import bench
    from paper_2011_05749_b200 import DsfftConfig, plan_cycles, rffast_batch, sfft_dt_batch
    from paper_2011_05749_b200.dsfft import dsfft_batch

    dev = torch.device("cuda", 0)
    S = SIGNALS[name]
    if name == "c2":
        n, k = 1 << 22, 1000
        x, _ = bench.synth_batch(n, k, "exact", list(range(S)), torch.complex128, dev)
        seeds = [bench.case_seed(n, k, "exact", 0, i) for i in range(S)]

        def call():
            sfft_dt_batch(x, k, 1024, 4, 15, "dt2", seeds=seeds)
    elif name in ("c3", "c3auto"):
        n, k = 511 * 512 * 513, 1000
        x, _ = bench.synth_batch(n, k, 20.0, list(range(S)), torch.complex128, dev, chunk=2)
        plans = [plan_cycles(n, k, "noisy", seed=bench.case_seed(n, k, 20.0, 0, i))
                 for i in range(S)]
        search = [p[1] for p in plans]
        factors = [511, 512, 513] if name == "c3" else list(plans[0][0].factors)

        def call():
            rffast_batch(x, k, factors, search)
    else:
        n, k, snr = 1 << 24, 4096, 20.0
        x, _ = bench.synth_batch(n, k, snr, list(range(S)), torch.complex64, dev, chunk=4)
        seeds = [bench.case_seed(n, k, snr, 0, i) for i in range(S)]
        if name == "c4dt3":
            def call():
                sfft_dt_batch(x, k, 4096, 4, 15, "dt3", seeds=seeds)
        else:
            cfgs = [DsfftConfig(mode="noisy", seed=s,
                                noise_std=float(np.sqrt(k * 10 ** (-snr / 10)))) for s in seeds]

            def call():
                dsfft_batch(x, k, cfgs)
    call()
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    call()
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()


def parse(csv_text):
    rows = list(csv.reader(io.StringIO(csv_text)))
    hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[hdr_i]
    col = {h: i for i, h in enumerate(hdr)}
    kernels = {}
    for r in rows[hdr_i + 1:]:
        if len(r) < len(hdr):
            continue
        kid = r[col["ID"]]
        ent = kernels.setdefault(kid, {"name": r[col["Kernel Name"]].split("(")[0]})
        v = r[col["Metric Value"]].replace(",", "")
        try:
            ent[r[col["Metric Name"]]] = float(v)
        except ValueError:
            pass
    return list(kernels.values())


def summarise(name, kernels):
    S = SIGNALS[name]
    tot_t = sum(k.get("gpu__time_duration.sum", 0.0) for k in kernels)
    flops = sum(k.get("sm__sass_thread_inst_executed_op_dadd_pred_on.sum", 0.0)
                + k.get("sm__sass_thread_inst_executed_op_dmul_pred_on.sum", 0.0)
                + 2 * k.get("sm__sass_thread_inst_executed_op_dfma_pred_on.sum", 0.0)
                for k in kernels)
    by = {}
    for k in kernels:
        e = by.setdefault(k["name"], {"launches": 0, "time_ns": 0.0, "fp64_flops": 0.0,
                                      "_pipe": 0.0, "_issue": 0.0})
        t = k.get("gpu__time_duration.sum", 0.0)
        e["launches"] += 1
        e["time_ns"] += t
        e["fp64_flops"] += (k.get("sm__sass_thread_inst_executed_op_dadd_pred_on.sum", 0.0)
                            + k.get("sm__sass_thread_inst_executed_op_dmul_pred_on.sum", 0.0)
                            + 2 * k.get("sm__sass_thread_inst_executed_op_dfma_pred_on.sum", 0.0))
        e["_pipe"] += t * k.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 0.0)
        e["_issue"] += t * k.get("sm__inst_issued.avg.pct_of_peak_sustained_active", 0.0)
    table = []
    for nm, e in by.items():
        table.append({"kernel": nm, "launches": e["launches"], "time_share": e["time_ns"] / tot_t,
                      "fp64_flops": e["fp64_flops"],
                      "fp64_pipe_pct": e["_pipe"] / e["time_ns"] if e["time_ns"] else 0.0,
                      "issue_pct": e["_issue"] / e["time_ns"] if e["time_ns"] else 0.0})
    table.sort(key=lambda r: -r["time_share"])
    dom = table[0] if table else {}
    return {"signals": S, "fp64_flops_per_signal": flops / S, "ncu_kernel_ms": tot_t / 1e6,
            "launches": len(kernels), "dominant_kernel": dom.get("kernel"),
            "dominant_fp64_pipe_pct": dom.get("fp64_pipe_pct"),
            "dominant_issue_pct": dom.get("issue_pct"), "kernels": table[:12]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c2,c3,c3auto,c4dt3,c4dsfft")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_pipes.json"))
    ap.add_argument("--child", default=None)
    args = ap.parse_args()
    if args.child:
        child(args.child)
        return
    out = {}
    if os.path.exists(args.out):
        with open(args.out) as fh:
            out = json.load(fh)
    for name in args.configs.split(","):
        cmd = ["ncu", "--profile-from-start", "off", "--clock-control", "none", "--csv",
               "--graph-profiling", "node",
               "--metrics", ",".join(METRICS), sys.executable, os.path.abspath(__file__),
               "--child", name]
        env = dict(os.environ)
        if name in ("c3", "c3auto"):
            # ncu does not profile the kernels inside the R-FFAST round graph's WHILE
            # body; the host-driven loop runs the same per-round kernels (its scan on a
            # grid instead of the persistent ticket grid)
            env["AFFT_PEEL_GRAPH"] = "0"
        p = subprocess.run(cmd, capture_output=True, text=True, env=env)
        if p.returncode != 0:
            print(p.stdout[-3000:], p.stderr[-3000:], file=sys.stderr)
            raise SystemExit(f"ncu failed for {name}")
        out[name] = summarise(name, parse(p.stdout))
        out[name]["command"] = " ".join(cmd[:-3]) + f" tools/ncu_pipes.py --child {name}"
        with open(args.out, "w") as fh:
            json.dump(out, fh, indent=1)
        print(name, json.dumps({k: v for k, v in out[name].items() if k != "kernels"}),
              flush=True)


if __name__ == "__main__":
    main()
