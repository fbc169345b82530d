"""Phase clocks of the CholeskyQR2 reconstruction kernel (cqr_recon_kernel, -DUTV_CQR_TRACE build:
UTV_TRACE=1 python -m paper_2408_05238_b200.build --force) for one 50000 x 64 sub-panel."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_05238_b200 as utv  # noqa: E402

h = utv.Handle(0)
for m, w in ((50000, 64), (50000, 256)):
    P0 = utv.colmajor_empty(m, w)
    P0.normal_()
    for _ in range(3):
        P = P0.clone()
        h.hqr(P)
    torch.cuda.synchronize()
    buf = (C.c_longlong * 16)()
    utv.lib().utv_debug_cqr_trace(buf)
    order = [0, 5, 1, 6, 2, 3, 7, 8, 4]
    names = ["load G2 + check", "chol(G2)", "R = R2 R1 (mm)", "Q_top row solves", "LU(sign)",
             "P/W writes, U', L^T", "T row solves", "M = U'R (mm) + write"]
    t = [buf[i] for i in order]
    print(f"{m}x{w} recon phases (us):", {names[i]: round((t[i + 1] - t[i]) / 1e3, 2) for i in range(len(names))},
          "total", round((t[-1] - t[0]) / 1e3, 2))
