"""K2' passes at n = 2^24 (diagnostic, for ncu launch lists): four dense transforms
(b = n, tau = 0) of a c64 or c128 signal; profile with --launch-skip 6 -c 3."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2011_05749_b200.bucketize import bucketize_device  # noqa: E402

dev = torch.device("cuda", 0)
n = 1 << 24
x = torch.randn(n, dtype=torch.complex128, device=dev)
if sys.argv[1:] == ["c64"]:
    x = x.to(torch.complex64)
for _ in range(4):
    bucketize_device(x, n, [0])
torch.cuda.synchronize()
