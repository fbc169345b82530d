"""Per-launch breakdown of one panel QR (utv_hqr) at randUTV's shapes, from the library's own
event profiler: the sub-panel kernels vs the inter-sub-panel GEMMs vs the T assembly."""
import csv
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_05238_b200 as utv  # noqa: E402

h = utv.Handle(0)
shapes = [(50000, 256), (200000, 256), (20000, 256), (2000, 256)]
if len(sys.argv) > 1:
    shapes = [tuple(int(x) for x in s.split("x")) for s in sys.argv[1:]]
os.makedirs("gpurun_out", exist_ok=True)
for m, w in shapes:
    P0 = utv.colmajor_empty(m, w)
    P0.normal_()
    P = P0.clone()
    for _ in range(3):
        P.copy_(P0)
        h.hqr(P)
    torch.cuda.synchronize()
    P.copy_(P0)
    h.profile(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(h.stream)
    h.hqr(P)
    e1.record(h.stream)
    torch.cuda.synchronize()
    path = f"gpurun_out/panel_{m}x{w}.csv"
    h.profile_dump(path)
    h.profile(False)
    rows = list(csv.DictReader(open(path)))
    tot = sum(float(r["ms"]) for r in rows)
    print(f"== hqr {m}x{w}: wall {e0.elapsed_time(e1):.3f} ms, sum of launches {tot:.3f} ms, {len(rows)} launches")
    for r in rows:
        print(f"  fam {r['family']} M={r['M']:>7s} N={r['N']:>5s} K={r['K']:>7s} tag={r['tag']:>6s} {float(r['ms'])*1e3:9.1f} us")
