"""Config-5 fused-kernel step time under AFFT_FUSED_ORDER 0/1/2 (diagnostic)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import bench  # noqa: E402
from ffast_modes import t  # noqa: E402
from paper_2011_05749_b200 import ffast_batch  # noqa: E402
from paper_2011_05749_b200.batch import ffast_workspace_bytes  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
dev = torch.device("cuda", 0)
x = torch.empty((S, bench.N_SIG), dtype=torch.complex64, device=dev)
bench.synth_signals(x, 0, dev)
ws = torch.empty(ffast_workspace_bytes(bench.N_SIG, 0, S, bench.FACTORS), dtype=torch.uint8,
                 device=dev)
os.environ["AFFT_FFAST_MODE"] = "0"
res = ffast_batch(x, bench.K, bench.FACTORS, workspace=ws)
ref = None
for rep in range(5):
    out = {}
    for order in ("0", "1", "2"):
        os.environ["AFFT_FUSED_ORDER"] = order
        out[order] = round(t(lambda: ffast_batch(x, bench.K, bench.FACTORS, workspace=ws, out=res), reps=15), 3)
        got = (res.count.clone(), res.pos.clone())
        if ref is None:
            ref = got
        assert torch.equal(ref[0], got[0]) and torch.equal(ref[1], got[1]), order
    print(rep, out, flush=True)
