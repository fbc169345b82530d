"""Summarise an `ncu --metrics gpu__time_duration.sum --csv --log-file` launch list by kernel."""
import collections
import csv
import re
import sys

lines = [ln for ln in open(sys.argv[1]) if ln.startswith('"')]
rows = list(csv.reader(lines))
hdr = rows[0]
ki, mi, ui, vi, si = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value", "Stream"))
scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3, "second": 1e3}
agg = collections.defaultdict(lambda: [0, 0.0])
tot, n = 0.0, 0
for r in rows[1:]:
    if r[mi] != "gpu__time_duration.sum":
        continue
    name = r[ki]
    short = re.sub(r"^void\s+", "", name).replace("<unnamed>::", "").replace("(anonymous namespace)::", "")
    short = re.sub(r"\(.*$", "", short)
    short = re.sub(r"<.*$", "", short)
    short = short.replace("utv::", "").replace("at::native::", "at::")
    ms = float(r[vi].replace(",", "")) * scale[r[ui]]
    agg[short][0] += 1
    agg[short][1] += ms
    tot += ms
    n += 1
print(f"{n} launches, {tot / 1e3:.3f} s total kernel time")
print(f"{'kernel':45s} {'launches':>8s} {'ms':>10s} {'share':>6s}")
for k, (c, ms) in sorted(agg.items(), key=lambda z: -z[1][1]):
    print(f"{k[:45]:45s} {c:8d} {ms:10.1f} {100 * ms / tot:5.1f}%")
