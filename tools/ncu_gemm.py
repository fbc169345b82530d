"""One launch of each main GEMM shape (for ncu --set full).  argv: n [shapes], shapes a comma list
of tn (sketch-type long K), nt (rank-256 update), nn (long-K Z = A'Y type); default tn,nt."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2408_05238_b200 as utv
h = utv.Handle(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
shapes = sys.argv[2].split(",") if len(sys.argv) > 2 else ["tn", "nt"]
def run(ta, tb, M, N, K, beta):
    A = utv.colmajor_empty(K if ta else M, M if ta else K); A.normal_()
    B = utv.colmajor_empty(N if tb else K, K if tb else N); B.normal_()
    Cm = utv.colmajor_empty(M, N); Cm.zero_()
    h.gemm(ta, tb, 1.0, A, B, beta, Cm); torch.cuda.synchronize()
for s in shapes:
    if s == "tn":
        run(True, False, n, 256, n, 0.0)      # sketch-type TN, long K
    elif s == "nt":
        run(False, True, n, n, 256, 1.0)      # rank-256 update NT
    elif s == "nn":
        run(False, False, n, 256, n, 0.0)     # Z = A' Y, X = A W_V: long K, A MN-major
