"""Summarise an ncu --metrics gpu__time_duration.sum launch-list CSV by kernel (diagnostic)."""
import collections
import csv
import sys

for path in sys.argv[1:]:
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        agg[r[ki]][0] += 1
        agg[r[ki]][1] += float(r[vi].replace(",", ""))
    tot = sum(v[1] for v in agg.values())
    print(path, "total %.3f ms" % (tot / 1e6))
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:8]:
        print("  %-60s %4d %9.3f ms %5.1f%%" % (k[:60], v[0], v[1] / 1e6, 100 * v[1] / tot))
