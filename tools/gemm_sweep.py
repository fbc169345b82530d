"""GEMM throughput at randUTV's cfg3 shapes (step 0 and mid-run), current build."""
import json, os, sys
import torch
sys.path.insert(0, ".")
import paper_2408_05238_b200 as utv
h = utv.Handle(0)
res = {}
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
    res[name] = {"ms": best * 1e3, "tflops": 2.0 * M * N * K / best / 1e12}
    print(os.environ.get("TAG", "auto"), name, res[name], flush=True)
    del A, B, Cm
for n in (50000, 25000):
    t_gemm(f"TN_{n}x256_K{n}", True, False, n, 256, n)
    t_gemm(f"NN_{n}x256_K{n}", False, False, n, 256, n)
    t_gemm(f"NT_update_{n}x{n}_K256", False, True, n, n, 256, beta=1.0)
    t_gemm(f"TN_256x{n}_K{n}", True, False, 256, n, n)
    t_gemm(f"NN_update_{n}x{n}_K256", False, False, n, n, 256, beta=1.0)
    t_gemm(f"NT_update_{n}x{n}_K512", False, True, n, n, 512, beta=1.0)
t_gemm("square_8192", False, False, 8192, 8192, 8192)
json.dump(res, open(f"gpurun_out/gemm_sweep_{os.environ.get('TAG', 'auto')}.json", "w"), indent=1)
