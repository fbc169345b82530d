"""Short-K update GEMMs (the fused K=2b and K=b updates) at cfg3 sizes under the current tile config."""
import json, os, sys
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
    print(os.environ.get("UTV_GEMM_CFG_SHORT", "d"), M, N, K, "%.2f ms %.2f TF/s" % (best * 1e3, 2.0 * M * N * K / best / 1e12), flush=True)
    del A, B, Cm
for n in (50000, 25000, 10000):
    t_gemm(False, True, n, n - 256, 512)
    t_gemm(False, True, n, n, 256)
