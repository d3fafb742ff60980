"""Summarise an ncu --csv launch list (gpu__time_duration.sum) by kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        nm = d["Kernel Name"].split("(")[0]
        agg[nm][0] += 1
        agg[nm][1] += float(d["Metric Value"])
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':60s} {'n':>5s} {'total ms':>10s} {'avg us':>10s} {'share':>6s}")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k[:60]:60s} {v[0]:5d} {v[1]/1e6:10.3f} {v[1]/v[0]/1e3:10.1f} {v[1]/tot:6.3f}")
print(f"total {tot/1e6:.3f} ms")
