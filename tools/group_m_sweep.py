"""Raster group height (UTV_GEMM_GROUP_M) vs the main cfg3 GEMM shapes: long-K sketch products
(TN n x 256 x n, NN n x 256 x n) and the K = 512 / 256 updates (NT)."""
import os, sys
import torch
sys.path.insert(0, ".")
import paper_2408_05238_b200 as utv
h = utv.Handle(0)
def t_gemm(ta, tb, M, N, K, beta=1.0, reps=3):
    A = utv.colmajor_empty(K if ta else M, M if ta else K); A.normal_()
    B = utv.colmajor_empty(N if tb else K, K if tb else N); B.normal_()
    Cm = utv.colmajor_empty(M, N); Cm.normal_()
    h.gemm(ta, tb, 1.0, A, B, beta, Cm); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(reps):
        e0.record(); h.gemm(ta, tb, 1.0, A, B, beta, Cm); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3)
    return 2.0 * M * N * K / best / 1e12
g = os.environ.get("UTV_GEMM_GROUP_M", "16")
res = []
res.append(t_gemm(True, False, 50000, 256, 50000, 0.0))
res.append(t_gemm(False, False, 50000, 256, 50000, 0.0))
res.append(t_gemm(False, True, 50000, 49744, 512))
res.append(t_gemm(False, True, 25000, 24744, 512))
res.append(t_gemm(False, True, 25000, 25000, 256))
print("group_m", g, " ".join("%.2f" % x for x in res), flush=True)
