"""Critical-path summary of a bench.py --profile-dump CSV (start_ms / stream columns): what the
main stream is busy with, the idle gaps on it, and the side stream's work."""
import collections
import csv
import sys

rows = list(csv.DictReader(open(sys.argv[1])))
fam = {"0": "gemm", "1": "panel", "2": "svd", "3": "sketch", "4": "solve", "5": "misc"}
main_id = rows[0]["stream"]


def cls(r):
    f = fam[r["family"]]
    if f != "gemm":
        return f
    K, fl = int(r["K"]), float(r["flops"])
    if fl < 4e9:
        return "gemm-small"
    return "gemm-longK" if K > 1024 else f"gemm-K{K}"


main = [r for r in rows if r["stream"] == main_id]
side = [r for r in rows if r["stream"] != main_id]
busy, cnt, flops = collections.Counter(), collections.Counter(), collections.Counter()
gaps, gapcnt = collections.Counter(), collections.Counter()
prev_end, prev = None, None
for r in main:
    s, d, c = float(r["start_ms"]), float(r["ms"]), cls(r)
    busy[c] += d; cnt[c] += 1; flops[c] += float(r["flops"])
    if prev_end is not None and s > prev_end:
        gaps[f"{prev} -> {c}"] += s - prev_end; gapcnt[f"{prev} -> {c}"] += 1
    prev_end, prev = s + d, c
end = max(float(r["start_ms"]) + float(r["ms"]) for r in rows)
print(f"timeline {end:.1f} ms; main stream {len(main)} launches, busy {sum(busy.values()):.1f} ms, "
      f"idle {sum(gaps.values()):.1f} ms; side stream {len(side)} launches")
print(f"{'main-stream class':18s} {'launches':>8s} {'ms':>10s} {'share':>6s} {'TF/s':>7s}")
for k, v in busy.most_common():
    tf = flops[k] / (v * 1e-3) / 1e12 if v > 0 and flops[k] > 0 else 0.0
    print(f"{k:18s} {cnt[k]:8d} {v:10.1f} {100 * v / end:5.1f}% {tf:7.2f}")
print("largest main-stream idle gaps (previous -> next launch):")
for k, v in gaps.most_common(5):
    print(f"  {k:32s} {gapcnt[k]:6d} {v:8.1f} ms")
sb = collections.Counter()
for r in side:
    sb[cls(r)] += float(r["ms"])
print("side stream (overlapped):", ", ".join(f"{k} {v:.1f} ms" for k, v in sb.most_common()))
