"""Time the wide (m < n) least-squares path (reading R21) on one GPU: randUTV of A^T with explicit
U', V'.  Usage: python tools/wide_bench.py [m n r b q]"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2408_05238_b200 as utv
import utv_inputs as gen

m, n, r, b, q = (int(x) for x in (sys.argv[1:6] if len(sys.argv) > 5 else (10000, 20000, 5000, 256, 2)))
At, Bm, X0 = gen.gp_torch(m, n, r, device="cuda", k=1)       # Gp recipe, column-major m x n (At = A^T rows)
A = At.t()
B = utv.colmajor(Bm)
X = utv.colmajor_empty(n, 1)
h = utv.Handle(0)
opts = utv.Opts(block=b, power_iters=q, tau=1e-10, seed=1)
for _ in range(2):
    rr = h.lstsq(A, B, X, opts)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(h.stream)
rr = h.lstsq(A, B, X, opts)
e1.record(h.stream)
torch.cuda.synchronize()
t = e0.elapsed_time(e1) / 1e3
err = (torch.linalg.norm(X - X0) / torch.linalg.norm(X0)).item()
print(f"wide m={m} n={n} r={r} b={b} q={q}: rank {rr}, {t:.3f} s, ||x - x0||/||x0|| = {err:.2e}", flush=True)
