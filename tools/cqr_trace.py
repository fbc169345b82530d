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
    t = [buf[i] for i in range(5)]
    names = ["", "G2 check + chol", "R, Q_top", "LU(sign)", "writes, T, M"]
    print(f"{m}x{w} recon phases (us):", {names[i]: round((t[i] - t[i - 1]) / 1e3, 2) for i in range(1, 5)},
          "total", round((t[4] - t[0]) / 1e3, 2))
