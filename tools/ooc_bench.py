"""Time the streamed (UTV_HOST_STREAMED) randUTV LS at a given size and resident-column cap."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2408_05238_b200 as utv
import utv_inputs as gen

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
caps = [int(c) for c in sys.argv[2:]] or [n, n // 2, 0]
h = utv.Handle(0)
At, Bm, X0 = gen.gp_torch(n, n, n // 2, device="cuda")
A0 = At.t().cpu()                       # column-major host copy (pageable)
B0 = utv.colmajor(Bm).cpu()
Ah = utv.colmajor_empty(n, n, device="cpu", pin_memory=True)
Bh = utv.colmajor_empty(n, 1, device="cpu", pin_memory=True)
X = utv.colmajor_empty(n, 1, device="cpu", pin_memory=True)
res = []
for cap in caps:
    os.environ["UTV_OOC_MAX_RESIDENT_COLS"] = str(cap)
    Ah.copy_(A0); Bh.copy_(B0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = h.lstsq(Ah, Bh, X, utv.Opts(block=256, power_iters=2, flags=utv.UTV_HOST_STREAMED))
    t = time.perf_counter() - t0
    st = h.stream_stats()
    err = ((X - X0.cpu()).norm() / X0.cpu().norm()).item()
    d = {"n": n, "cap": cap, "s": t, "rank": r, "rel_err_x0": err, **st,
         "link_GBps": (st["h2d_bytes"] + st["d2h_bytes"]) / t / 1e9}
    print(json.dumps(d), flush=True)
    res.append(d)
json.dump(res, open(f"gpurun_out/ooc_bench_{n}.json", "w"), indent=1)
