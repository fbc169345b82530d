"""GEMM correctness at randUTV's large shapes (TMA and cp.async paths) against torch FP64 matmul."""
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_2408_05238_b200 as utv

h = utv.Handle(0)
torch.manual_seed(0)
tag = os.environ.get("UTV_GEMM_TMA", "1") + "/" + os.environ.get("UTV_GEMM_CFG_SHORT", "d")


def view(rows, cols, ld_pad=0, off=0):
    base = utv.colmajor_empty(rows + ld_pad + off, cols)
    base.normal_()
    return base[off:off + rows]


def check(name, ta, tb, M, N, K, beta=0.0, pad=0, off=0):
    A = view(K if ta else M, M if ta else K, pad, off)
    B = view(N if tb else K, K if tb else N, pad, off)
    Cm = view(M, N, pad, off)
    C0 = Cm.clone()
    h.gemm(ta, tb, -1.0, A, B, beta, Cm)
    ref = -((A.t() if ta else A) @ (B.t() if tb else B)) + beta * C0
    D = (Cm - ref).abs() > 1e-10 * ref.abs().max()
    err = ((Cm - ref).abs().max() / ref.abs().max()).item()
    if D.any():
        idx = D.nonzero()
        rows = torch.unique(idx[:, 0] // 128)
        cols = torch.unique(idx[:, 1] // 64)
        print(f"   bad: {D.sum().item()} of {D.numel()}; tile-rows {rows[:12].tolist()} ({rows.numel()}), "
              f"tile-cols(64) {cols[:12].tolist()} ({cols.numel()}); first {idx[:4].tolist()}", flush=True)
    print(f"TMA={tag} {name:28s} M={M} N={N} K={K} beta={beta} pad={pad} off={off}: max rel err {err:.2e}",
          "FAIL" if err > 1e-12 else "ok", flush=True)


for n in [int(a) for a in sys.argv[1:]] or (20000, 19744):
    check("sketch TN", True, False, n, 256, n)
    check("power NN", False, False, n, 256, n)
    check("left P TN", True, False, 256, n, n)
    check("update NT K=512", False, True, n, n, 512, beta=1.0)
    check("update NT K=256", False, True, n, n, 256, beta=1.0)
    check("update NN K=256", False, False, n, n, 256, beta=1.0)
check("narrow TN (P_r^T W)", True, False, 224, 32, 50000)
check("narrow NN", False, False, 20000, 32, 256, beta=1.0)
check("narrow NT k=1", False, True, 20000, 1, 256, beta=1.0)
check("narrow TN k=16", True, False, 256, 16, 20000)
check("sub-view NT", False, True, 7000, 6000, 512, beta=1.0, pad=256, off=256)
check("sub-view TN", True, False, 6000, 256, 7000, pad=256, off=256)
check("sub-view NN", False, False, 6000, 256, 7000, beta=1.0, pad=2, off=2)
check("sub-view TT", True, True, 3000, 2000, 1500, beta=1.0, pad=2, off=2)
