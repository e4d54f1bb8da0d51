"""Component timing of the config-5 FFAST step (diagnostic): norm stream alone,
decode alone (eps precomputed), fused single kernel, pipelined two-stream."""

import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2011_05749_b200 import _lib, ffast_batch  # noqa: E402
from paper_2011_05749_b200.batch import ffast_workspace_bytes  # noqa: E402


def t(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    S = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
    dev = torch.device("cuda", 0)
    x = torch.empty((S, bench.N_SIG), dtype=torch.complex64, device=dev)
    bench.synth_signals(x, 0, dev)
    lib = _lib.load()
    nparts = lib.afft_sumsq_parts(bench.N_SIG, 0)
    part = torch.empty((S, nparts), dtype=torch.float64, device=dev)
    eps = torch.empty(S, dtype=torch.float64, device=dev)
    sp = torch.cuda.current_stream().cuda_stream
    ms_norm = t(lambda: lib.afft_sumsq(x.data_ptr(), 0, bench.N_SIG, S, bench.N_SIG,
                                       part.data_ptr(), sp))
    ws = torch.empty(ffast_workspace_bytes(bench.N_SIG, 0, S, bench.FACTORS), dtype=torch.uint8,
                     device=dev)
    res = ffast_batch(x, bench.K, bench.FACTORS, workspace=ws)
    out = {}
    for mode in ("0", "1", "2", "3"):
        os.environ["AFFT_FFAST_MODE"] = mode
        out[mode] = t(lambda: ffast_batch(x, bench.K, bench.FACTORS, workspace=ws, out=res))
    import ctypes
    fb, nc = _lib.host_i64(bench.FACTORS)
    blk, sm = ctypes.c_int32(0), ctypes.c_int32(0)
    lib.afft_ffast_occupancy(bench.N_SIG, fb, nc, ctypes.byref(blk), ctypes.byref(sm))
    print(f"fused kernel: {blk.value} CTAs/SM, {sm.value} B dynamic smem")
    for rep in range(2):
        for mode in ("0", "1", "2", "3"):
            os.environ["AFFT_FFAST_MODE"] = mode
            out[mode] = t(lambda: ffast_batch(x, bench.K, bench.FACTORS, workspace=ws, out=res))
        print(rep, {k: round(v, 3) for k, v in out.items()})
    os.environ["AFFT_FFAST_MODE"] = "2"
    for per_sm in ("1", "2", "3"):
        os.environ["AFFT_DECODE_CTAS_PER_SM"] = per_sm
        print("pipelined, decode CTAs/SM", per_sm,
              round(t(lambda: ffast_batch(x, bench.K, bench.FACTORS, workspace=ws, out=res)), 3))
    del os.environ["AFFT_DECODE_CTAS_PER_SM"]
    print("(stream loads: AFFT_STREAM_NO_ALLOCATE =", os.environ.get("AFFT_STREAM_NO_ALLOCATE", "1"), ")")
    gb = S * bench.SIGNAL_BYTES / 1e6
    print(f"signals {S}: norm alone {ms_norm:.3f} ms ({gb / ms_norm:.0f} GB/s); "
          f"fused(mode0) {out['0']:.3f}; prepass+decode(mode1) {out['1']:.3f} "
          f"(decode ~{out['1'] - ms_norm:.3f}); pipelined(mode2) {out['2']:.3f} ms; "
          f"split roles(mode3) {out['3']:.3f} ms")


if __name__ == "__main__":
    main()
