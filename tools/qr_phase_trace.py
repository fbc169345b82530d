"""Per-column phase clocks of the cooperative panel kernel (CTA 0), from a -DUTV_QR_TRACE build:
phases 0 start -> 3 block reduce + partial store -> 4 grid barrier -> 1 partial sums + pivot row
-> 2 dlarfg / w / s -> (row update) -> next column's 0.  Usage (GPU box):
  UTV_TRACE=1 python -c 'from paper_2408_05238_b200 import build as b; b.build(force=True)'
  python tools/qr_phase_trace.py 50000"""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2408_05238_b200 as utv  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 50000
h = utv.Handle(0)
L = utv.lib()
P0 = utv.colmajor_empty(m, 32)
P0.normal_()
for _ in range(3):
    P = P0.clone()
    h.hqr(P)
torch.cuda.synchronize()
buf = (ctypes.c_longlong * 1024)()
L.utv_debug_qr_trace(buf)
t = np.array(buf[:512]).reshape(64, 8)[:32]
ghz = 1.965
seg = {"reduce+store (0->3)": t[:, 3] - t[:, 0], "barrier (3->4)": t[:, 4] - t[:, 3],
       "partials (4->1)": t[:, 1] - t[:, 4], "dlarfg (1->2)": t[:, 2] - t[:, 1],
       "row update (2->next 0)": np.append(t[1:, 0] - t[:-1, 2], np.nan)}
tot = (t[31, 2] - t[0, 0]) / 31
print(f"m={m}: per column {tot / ghz / 1e3:.2f} us (CTA 0 clocks @ {ghz} GHz)")
for k, v in seg.items():
    print(f"  {k:24s} {np.nanmedian(v) / ghz / 1e3:6.2f} us")
