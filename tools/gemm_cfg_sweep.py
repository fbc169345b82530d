import sys, torch
sys.path.insert(0, ".")
import paper_2408_05238_b200 as utv
h = utv.Handle(0)
def t_gemm(M, N, K, cfg, reps=3):
    A = utv.colmajor_empty(M, K); A.normal_()
    B = utv.colmajor_empty(N, K); B.normal_()
    Cm = utv.colmajor_empty(M, N); Cm.normal_()
    with utv.tuned(utv.UTV_TUNE_GEMM_CFG, cfg):
        h.gemm(False, True, -1.0, A, B, 1.0, Cm); torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        best = 1e9
        for _ in range(reps):
            e0.record(); h.gemm(False, True, -1.0, A, B, 1.0, Cm); e1.record(); torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1) / 1e3)
    print(f"cfg {cfg} {M}x{N}x{K}: {best*1e3:.2f} ms {2.0*M*N*K/best/1e12:.2f} TF/s", flush=True)
for (M, N, K) in ((30000, 29744, 512), (30000, 30000, 256)):
    for cfg in (5, 0, 1, 2, 3, 4):
        t_gemm(M, N, K, cfg)
