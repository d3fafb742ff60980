"""Per-launch duration and DRAM bytes of every CTA-pair-engine launch of one C5 solve, from an ncu
metrics CSV (ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
-k regex:pair_power_kernel --csv python scripts/one_solve.py c5).  In launch order: mode-1 sketch,
5 power steps, shrink, then modes 2 and 3 (power steps, shrink).  HBM fraction against
MEASURED_PEAKS.json's copy bandwidth.  ncu serialises launches with a cold L2, so op2's re-reads
in the power steps partly come from DRAM here."""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
iid, iname, imet, ival = hdr.index("ID"), hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
iunit = hdr.index("Metric Unit")
SCALE = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0,
         "byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0}
per = {}
for r in rows[1:]:
    if "pair_power" not in r[iname]:
        continue
    per.setdefault(int(r[iid]), {})[r[imet]] = float(r[ival].replace(",", "")) * SCALE.get(r[iunit], 1.0)
hbm = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
# modes 2 and 3 sketch on tc_op2 (m < RTK_FUSED_SKETCH_MIN = 1e5), not on the pair engine
labels = ["m1 sketch"] + [f"m1 power {i}" for i in range(1, 6)] + ["m1 shrink"] + \
    [f"m2 power {i}" for i in range(1, 6)] + ["m2 shrink"] + [f"m3 power {i}" for i in range(1, 6)] + ["m3 shrink"]
print(f"| launch | ms | DRAM read GB | DRAM write GB | GB/s | of {hbm:.0f} GB/s |")
print("|---|---|---|---|---|---|")
for n, (k, m) in enumerate(sorted(per.items())):
    ms = m.get("gpu__time_duration.sum", 0)
    rd = m.get("dram__bytes_read.sum", 0)
    wr = m.get("dram__bytes_write.sum", 0)
    lab = labels[n] if n < len(labels) else str(n)
    bw = (rd + wr) / ms * 1e3 if ms else 0
    print(f"| {lab} | {ms:.3f} | {rd:.3f} | {wr:.3f} | {bw:.0f} | {bw / hbm:.2f} |")
