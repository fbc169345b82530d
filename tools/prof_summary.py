"""Summarise a utv_profile_dump CSV: GEMM time by shape class, other families."""
import csv, sys, collections
rows = list(csv.DictReader(open(sys.argv[1])))
fam = {0: "gemm", 1: "panel", 2: "svd", 3: "sketch", 4: "solve", 5: "misc"}
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for r in rows:
    f = fam[int(r["family"])]
    ms, fl = float(r["ms"]), float(r["flops"])
    if f == "gemm":
        M, N, K, tag = int(r["M"]), int(r["N"]), int(r["K"]), int(r["tag"])
        ta, tb, cfg, sp = tag & 1, (tag >> 1) & 1, (tag >> 2) & 63, tag >> 8
        kind = ("T" if ta else "N") + ("T" if tb else "N")
        small = M * N * K < 2e9
        if small: key = f"gemm small (<4 GF) {kind}"
        elif K <= 1024: key = f"gemm shortK K={K if K in (256, 512) else 'other'} {kind}"
        elif min(M, N) <= 512: key = f"gemm longK skinny {kind}"
        else: key = f"gemm other {kind}"
    else:
        key = f
    a = agg[key]; a[0] += 1; a[1] += ms; a[2] += fl
tot = sum(v[1] for v in agg.values())
print(f"{'class':40s} {'calls':>7s} {'ms':>10s} {'share':>6s} {'TF/s':>7s}")
for k, (n, ms, fl) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:40s} {n:7d} {ms:10.1f} {100*ms/tot:5.1f}% {fl/ms/1e9 if ms > 0 else 0:7.2f}")
