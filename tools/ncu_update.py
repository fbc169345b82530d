"""One fused K = 2b trailing-update GEMM (NT, beta = 1) at cfg3 step-0 size, for ncu --set full."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2408_05238_b200 as utv
h = utv.Handle(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 50000
K = int(sys.argv[2]) if len(sys.argv) > 2 else 512
A = utv.colmajor_empty(n, K).normal_()
B = utv.colmajor_empty(n - 256, K).normal_()
Cm = utv.colmajor_empty(n, n - 256).normal_()
h.gemm(False, True, -1.0, A, B, 1.0, Cm)
torch.cuda.synchronize()
