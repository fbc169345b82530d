"""Measure the FP64 roofline denominators on the B200 box (measurement only).

DMMA / DFMA microbenchmarks (tools/fp64_peak.cu) and cuBLAS DGEMM through
torch.matmul on float64 (a library ceiling, never on the product path).
"""
import json, subprocess, sys, time, os
import torch

out = {}
r = subprocess.run([os.path.join(os.path.dirname(__file__), "fp64_peak")], capture_output=True, text=True)
print(r.stdout, r.stderr)
try:
    out["microbench"] = json.loads(r.stdout.strip().splitlines()[-1])
except Exception as e:  # keep going
    out["microbench_error"] = str(e)

dev = torch.device("cuda:0")
for n in (8192, 16384):
    a = torch.randn(n, n, dtype=torch.float64, device=dev)
    b = torch.randn(n, n, dtype=torch.float64, device=dev)
    c = a @ b
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); c = a @ b; e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3)
    out[f"cublas_dgemm_{n}_burst_tflops"] = 2 * n**3 / best / 1e12
# sustained 8192^3 for ~4 s
n = 8192
a = torch.randn(n, n, dtype=torch.float64, device=dev); b = torch.randn(n, n, dtype=torch.float64, device=dev)
torch.cuda.synchronize(); t0 = time.time(); cnt = 0
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
while time.time() - t0 < 4.0:
    c = a @ b; cnt += 1
    if cnt % 4 == 0: torch.cuda.synchronize()
e1.record(); torch.cuda.synchronize()
out["cublas_dgemm_8192_sustained_tflops"] = 2 * n**3 * cnt / (e0.elapsed_time(e1) / 1e3) / 1e12
# rank-256 update shape (the trailing update)
m = 50000; k = 256
try:
    A = torch.randn(m, m, dtype=torch.float64, device=dev)
    X = torch.randn(m, k, dtype=torch.float64, device=dev)
    W = torch.randn(m, k, dtype=torch.float64, device=dev)
    A.addmm_(X, W.t(), alpha=-1.0); torch.cuda.synchronize()
    e0.record(); A.addmm_(X, W.t(), alpha=-1.0); e1.record(); torch.cuda.synchronize()
    out["cublas_rank256_update_50000_tflops"] = 2 * m * m * k / (e0.elapsed_time(e1) / 1e3) / 1e12
    e0.record(); Y = A.t() @ X; e1.record(); torch.cuda.synchronize()
    out["cublas_tn_50000x256_K50000_tflops"] = 2 * m * m * k / (e0.elapsed_time(e1) / 1e3) / 1e12
    del A
except Exception as e:
    out["rank256_error"] = str(e)
# HBM copy
x = torch.empty(1 << 30, dtype=torch.float64, device=dev); y = torch.empty_like(x)
y.copy_(x); torch.cuda.synchronize(); best = 1e9
for _ in range(5):
    e0.record(); y.copy_(x); e1.record(); torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1) / 1e3)
out["hbm_copy_gbs"] = 2 * x.numel() * 8 / best / 1e9
# pinned host <-> device
h = torch.empty(1 << 28, dtype=torch.float64, pin_memory=True)
d = torch.empty(1 << 28, dtype=torch.float64, device=dev)
d.copy_(h, non_blocking=True); torch.cuda.synchronize()
e0.record(); d.copy_(h, non_blocking=True); e1.record(); torch.cuda.synchronize()
out["h2d_pinned_gbs"] = h.numel() * 8 / (e0.elapsed_time(e1) / 1e3) / 1e9
e0.record(); h.copy_(d, non_blocking=True); e1.record(); torch.cuda.synchronize()
out["d2h_pinned_gbs"] = h.numel() * 8 / (e0.elapsed_time(e1) / 1e3) / 1e9
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/fp64_peaks.json", "w"), indent=1)
print(json.dumps(out, indent=1))
