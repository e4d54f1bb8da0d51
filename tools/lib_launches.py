"""Summarise an ncu --csv launch list, library kernels only (torch synthesis kernels
dropped): time per kernel name (ns -> ms), share, mean FP64-pipe % when captured."""
import collections
import csv
import sys

LIB = ("afft", "gfft", "gstockham", "gather_dft", "ffast_", "peel", "noisy", "dt_", "alias",
       "active_", "sumsq", "twiddle", "rows_", "coset", "dsfft", "search_list", "scan_counts",
       "selective", "truncate", "median", "robust", "node_energy", "count_multi")


def main(path, top=12):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ki, mn, mv, mu = (h.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    ms = collections.defaultdict(float)
    fp = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows[1:]:
        name = r[ki]
        if not any(k in name for k in LIB):
            continue
        key = name.split("(")[0][:70]
        v = float(r[mv].replace(",", ""))
        if r[mn] == "gpu__time_duration.sum":
            scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0}.get(r[mu], 1e-6)
            ms[key] += v * scale
            cnt[key] += 1
        elif "fp64" in r[mn]:
            fp[key] += v
    tot = sum(ms.values())
    print(f"{path}: library kernels {tot:.3f} ms")
    for k, v in sorted(ms.items(), key=lambda kv: -kv[1])[:top]:
        f = f"  FP64 {fp[k] / cnt[k]:.0f}%" if k in fp else ""
        print(f"  {k:70s} {cnt[k]:4d} {v:8.3f} ms {100 * v / tot:5.1f}%{f}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 12)
