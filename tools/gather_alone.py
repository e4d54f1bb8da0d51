"""The config-5 gather + 9 DFTs on their own (afft_build_graph -> gather_dft_kernel),
SURVEY §8(d): sectors fetched / kernel time / HBM peak, beside the full-path figure.

    python tools/gather_alone.py [signals]      (then the same under ncu for sectors)
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2011_05749_b200 import _lib  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
dev = torch.device("cuda", 0)
x = torch.empty((S, bench.N_SIG), dtype=torch.complex64, device=dev)
bench.synth_signals(x, 0, dev)
nodes = sum(bench.FACTORS)
out = torch.empty((S, nodes, 3), dtype=torch.complex128, device=dev)
lib = _lib.load()
fb, nc = _lib.host_i64(bench.FACTORS)
sb, ns = _lib.host_i64([0, 1, 2])
sp = torch.cuda.current_stream().cuda_stream


def run():
    _lib.check(lib.afft_build_graph(x.data_ptr(), 0, bench.N_SIG, S, bench.N_SIG, fb, nc, sb, ns,
                                    out.data_ptr(), sp), "build_graph")


run()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 10
a.record()
for _ in range(reps):
    run()
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / reps
alg = 22400 * S  # 22.5 KB of 32-B gather sectors per signal (1,152 samples)
print(json.dumps({"signals": S, "ms": ms, "us_per_signal": ms * 1e3 / S,
                  "sector_bytes_algorithmic": alg, "gbps_algorithmic": alg / ms / 1e6,
                  "frac_of_hbm_peak": alg / ms / 1e6 / bench.load_peaks()[0]}))
