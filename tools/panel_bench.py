"""Latency of the panel QR (utv_hqr) and the small SVD (utv_svd_small) at randUTV's shapes."""
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
for m, w in ((50000, 256), (20000, 256), (2000, 256), (256, 256), (50000, 32)):
    P0 = utv.colmajor_empty(m, w); P0.normal_()
    P = P0.clone()
    def f():
        P.copy_(P0); h.hqr(P)
    res[f"hqr_{m}x{w}_ms"] = timeit(f)
    print(f"hqr {m}x{w}", res[f"hqr_{m}x{w}_ms"], "ms", flush=True)
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
