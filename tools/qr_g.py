"""Panel-QR latency vs the number of cooperative CTAs (UTV_QR_MAXCTAS)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2408_05238_b200 as utv

h = utv.Handle(0)
for m, w in ((50000, 32), (50000, 256), (20000, 32)):
    P0 = utv.colmajor_empty(m, w)
    P0.normal_()
    P = P0.clone()
    h.hqr(P)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(5):
        P.copy_(P0)
        e0.record()
        h.hqr(P)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(sys.argv[1] if len(sys.argv) > 1 else "", m, w, round(best, 3), "ms", flush=True)
