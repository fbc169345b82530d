"""Latency of the panel QR (utv_hqr) at randUTV's shapes, per panel algorithm (utv_tune
UTV_TUNE_QR_CHOLQR: 0 automatic = CholeskyQR2 on tall sub-panels, 1 = Householder kernels only),
and of the small SVD (utv_svd_small).  Writes gpurun_out/panel_bench.json."""
import sys, json
import torch
sys.path.insert(0, ".")
import paper_2408_05238_b200 as utv
h = utv.Handle(0)
res = {}
def timeit(f, reps=5):
    f(); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(reps):
        e0.record(); f(); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best
shapes = ((200000, 256), (100000, 256), (50000, 256), (20000, 256), (5000, 256), (2048, 256), (1024, 256),
          (256, 256), (50000, 32))
for mode, name in ((1, "householder"), (0, "auto")):
    with utv.tuned(utv.UTV_TUNE_QR_CHOLQR, mode):
        for m, w in shapes:
            P0 = utv.colmajor_empty(m, w); P0.normal_()
            P = P0.clone()
            def f():
                P.copy_(P0); h.hqr(P)
            key = f"hqr_{name}_{m}x{w}_ms"
            res[key] = timeit(f)
            print(key, round(res[key], 4), flush=True)
torch.manual_seed(5)
R = torch.triu(torch.randn(256, 256, dtype=torch.float64, device="cuda")).t().contiguous().t()
def g():
    h.svd_small(R)
res["svd_small_256_ms"] = timeit(g)
sw = h.svd_small(R)[3]
res["svd_small_256_sweeps"] = sw
print("svd_small 256", res["svd_small_256_ms"], "ms, sweeps", sw, "->", res["svd_small_256_ms"] / sw, "ms per sweep", flush=True)
json.dump(res, open("gpurun_out/panel_bench.json", "w"), indent=1)
if len(sys.argv) > 1:   # profiling mode: one more call of each
    P.copy_(P0); h.hqr(P); h.svd_small(R); torch.cuda.synchronize()
