"""Debug: GPU randUTV T, V vs the oracle's, element by element (sign pattern of differences)."""
import sys
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np
import torch
import oracle
import utv_inputs as gen
import paper_2408_05238_b200 as utv


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.float64).T)).cuda().t()


h = utv.Handle(0)
for (m, n, r, b, q, tail) in [(300, 260, 100, 32, 1, 1e-9), (300, 260, 100, 32, 1, 0.0), (200, 180, 64, 64, 0, 1e-9)]:
    rng = np.random.default_rng(50 + r)
    A = gen.GdMatrix(m, n, r, alpha=2.0, seed=50 + r).A + tail * rng.standard_normal((m, n))
    Ad = dev(A); V = dev(np.zeros((n, n)))
    rk = h.factor(Ad, V=V, opts=utv.Opts(block=b, power_iters=q, tau=1e-7, seed=6))
    T, Vg = Ad.cpu().numpy(), V.cpu().numpy()
    out = oracle.randutv(A, b, q, seed=6)
    To, Vo = out["T"], out["V"]
    print(m, n, r, b, q, tail, "rank", rk, oracle.rank(To, 1e-7))
    for j0 in range(0, n, b):
        j1 = min(n, j0 + b)
        dv = np.abs(Vg[:, j0:j1] - Vo[:, j0:j1]).max(axis=0)
        sv = np.abs(Vg[:, j0:j1] + Vo[:, j0:j1]).max(axis=0)
        print("  blk", j0, "V same", int((dv < 1e-8).sum()), "V negated", int((sv < 1e-8).sum()), "of", j1 - j0,
              "Tdiag err", np.abs(np.diag(T)[j0:j1] - np.diag(To)[j0:j1]).max(), flush=True)
    d = np.abs(T[:r, :] - To[:r, :])
    print("  T[:r, :r] err", d[:, :r].max(), "T[:r, r:] err", d[:, r:].max())
