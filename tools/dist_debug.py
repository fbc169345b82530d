"""Debug the in-process multi-rank path: per-block diag(T) of P ranks vs the single-GPU path."""
import sys
import threading

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2408_05238_b200 as utv
import utv_inputs as gen
from paper_2408_05238_b200 import dist as D

P = int(sys.argv[1]) if len(sys.argv) > 1 else 2
m, n, r, b, q = 600, 600, 300, 64, 1
M = gen.GpMatrix(m, n, r, seed=7)
B, _ = M.known_rhs(k=1)
Ad = torch.from_numpy(np.ascontiguousarray(M.A.T)).cuda().t()
Bd = torch.from_numpy(np.ascontiguousarray(B.reshape(m, 1).T)).cuda().t()

A1 = utv.colmajor(Ad.clone()); B1 = Bd.clone()
X1, r1 = utv.lstsq(A1, B1, utv.Opts(block=b, power_iters=q, seed=3))
d1 = torch.diagonal(A1).cpu().numpy()

hs = utv.local_group(P)
shards = [utv.colmajor(D.scatter_columns(Ad, b, P, p).clone()) for p in range(P)]
Bs = [Bd.clone() for _ in range(P)]
Xs = [utv.colmajor_empty(n, 1) for _ in range(P)]
torch.cuda.synchronize()
res = [None] * P


def work(p):
    try:
        res[p] = hs[p].lstsq(shards[p], Bs[p], Xs[p], utv.Opts(block=b, power_iters=q, seed=3))
    except Exception as e:  # noqa
        res[p] = repr(e)


ts = [threading.Thread(target=work, args=(p,)) for p in range(P)]
[t.start() for t in ts]
[t.join(120) for t in ts]
print("alive:", [t.is_alive() for t in ts], "ranks:", res, "single:", r1, flush=True)
torch.cuda.synchronize()
T = D.gather_columns(shards, n, b)
dP = torch.diagonal(T).cpu().numpy()
for blk in range(n // b):
    e = np.max(np.abs(dP[blk * b:(blk + 1) * b] - d1[blk * b:(blk + 1) * b])) / np.max(np.abs(d1))
    print(f"block {blk}: max |d_P - d_1| / max d = {e:.2e}")
for p in range(P):
    print("rank", p, "x vs single:", (Xs[p] - X1).norm().item() / X1.norm().item())
