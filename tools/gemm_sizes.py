"""GEMM efficiency across the trailing sizes a cfg3 run visits (sketch TN/NN, fused K=512 update)."""
import json, sys
import torch
sys.path.insert(0, ".")
import paper_2408_05238_b200 as utv
h = utv.Handle(0)
res = []
def t_gemm(name, ta, tb, M, N, K, beta=0.0, reps=3):
    A = utv.colmajor_empty(K if ta else M, M if ta else K); A.normal_()
    B = utv.colmajor_empty(N if tb else K, K if tb else N); B.normal_()
    Cm = utv.colmajor_empty(M, N); Cm.normal_()
    h.gemm(ta, tb, 1.0, A, B, beta, Cm); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(reps):
        e0.record(); h.gemm(ta, tb, 1.0, A, B, beta, Cm); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3)
    d = {"name": name, "M": M, "N": N, "K": K, "ms": best * 1e3, "tflops": 2.0 * M * N * K / best / 1e12}
    print(json.dumps(d), flush=True); res.append(d)
    del A, B, Cm
for n in [int(a) for a in sys.argv[1:]] or (50000, 40000, 30000, 20000, 12000, 8000, 5000, 3000):
    t_gemm("TN", True, False, n, 256, n)
    t_gemm("NN", False, False, n, 256, n)
    t_gemm("NT_K512", False, True, n, n - 256, 512, beta=1.0)
json.dump(res, open("gpurun_out/gemm_sizes.json", "w"), indent=1)
