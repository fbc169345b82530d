"""Time the DMMA GEMM at randUTV's shapes (cfg3 step 0) and a small end-to-end lstsq."""
import sys, time, json
import torch
sys.path.insert(0, ".")
import paper_2408_05238_b200 as utv

h = utv.Handle(0)
dev = "cuda:0"
res = {}
def t_gemm(name, ta, tb, M, N, K, beta=0.0, reps=3):
    A = utv.colmajor_empty(K if ta else M, M if ta else K); A.normal_()
    B = utv.colmajor_empty(N if tb else K, K if tb else N); B.normal_()
    Cm = utv.colmajor_empty(M, N); Cm.zero_()
    h.gemm(ta, tb, 1.0, A, B, beta, Cm); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(reps):
        e0.record(); h.gemm(ta, tb, 1.0, A, B, beta, Cm); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3)
    res[name] = {"ms": best * 1e3, "tflops": 2.0 * M * N * K / best / 1e12}
    print(name, res[name], flush=True)
    del A, B, Cm
n = int(sys.argv[1]) if len(sys.argv) > 1 else 50000
t_gemm("sketch_TN_n'x256_K=m'", True, False, n, 256, n)
t_gemm("power_NN_m'x256_K=n'", False, False, n, 256, n)
t_gemm("rank256_update_NT", False, True, n, n, 256, beta=1.0)
t_gemm("left_P_TN_256xn'", True, False, 256, n, n)
t_gemm("square_8192", False, False, 8192, 8192, 8192)
# end-to-end small lstsq timing
import utv_inputs as gen
for nn, b in ((4096, 256), (8192, 256)):
    At, Bm, X0 = gen.gp_torch(nn, nn, nn // 2, device=dev)
    A = At.t(); B = utv.colmajor(Bm)
    A0 = A.clone(); B0 = B.clone()
    X, r = utv.lstsq(A.clone(), B.clone(), utv.Opts(block=b, power_iters=2)); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    Ac, Bc = utv.colmajor(A0.clone()), B0.clone()
    e0.record(); X, r = utv.lstsq(Ac, Bc, utv.Opts(block=b, power_iters=2)); e1.record(); torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 1e3
    F = (18 + 8) / 3 * nn ** 3
    err = ((X - X0).norm() / X0.norm()).item()
    res[f"lstsq_{nn}"] = {"s": t, "tflops_alg": F / t / 1e12, "rank": r, "rel_err_x0": err}
    print(f"lstsq_{nn}", res[f"lstsq_{nn}"], flush=True)
json.dump(res, open("gpurun_out/gemm_bench.json", "w"), indent=1)
