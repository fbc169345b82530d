"""Debug: GPU nullify vs a numpy emulation applied to the GPU's own pre-nullify T, V."""
import sys
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np
import torch
import oracle
import utv_inputs as gen
import paper_2408_05238_b200 as utv


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.float64).T)).cuda().t()


def emu(T, V, r, b):
    T = T.copy(); V = V.copy(); n = V.shape[0]; nz = n - r; i1 = r
    while i1 > 0:
        i0 = max(0, i1 - b); bw = i1 - i0
        S = np.hstack([T[i0:i1, i0:i1], T[i0:i1, r:n]])
        J = np.eye(bw)[::-1]; D = np.eye(bw + nz); D[:bw, :bw] = J
        P, tau, Tz = oracle.hqr(D @ S.T @ J)
        W = np.tril(P[:, :bw], -1); W[np.arange(bw), np.arange(bw)] = 1
        C = np.eye(bw + nz) - (D @ W) @ Tz @ (D @ W).T
        cols = list(range(i0, i1)) + list(range(r, n))
        T[i0:i1, i0:i1] = J @ np.triu(P[:bw, :bw]).T @ J; T[i0:i1, r:n] = 0
        T[:i0][:, cols] = T[:i0][:, cols] @ C
        V[:, cols] = V[:, cols] @ C
        i1 = i0
    return T, V


h = utv.Handle(0)
for (m, n, r, b, q) in [(300, 260, 100, 32, 1), (200, 180, 64, 64, 0), (150, 150, 149, 16, 1), (120, 100, 7, 32, 2)]:
    rng = np.random.default_rng(50 + r)
    A = gen.GdMatrix(m, n, r, alpha=2.0, seed=50 + r).A + 1e-9 * rng.standard_normal((m, n))
    res = []
    for fl in (0, utv.UTV_NULLIFY_T12):
        Ad = dev(A); V = dev(np.zeros((n, n)))
        rk = h.factor(Ad, V=V, opts=utv.Opts(block=b, power_iters=q, tau=1e-7, seed=6, flags=fl))
        res.append((Ad.cpu().numpy(), V.cpu().numpy(), rk))
    (T0, V0, r0), (T1, V1, r1) = res
    Te, Ve = emu(T0, V0, r0, b)
    d = np.abs(T1[:r0, :] - Te[:r0, :])
    i, j = np.unravel_index(np.argmax(d), d.shape)
    print(m, n, r, b, "rank", r0, r1, "T err", d.max(), "at", (i, j), "V err", np.abs(V1 - Ve)[:, :r0].max(), flush=True)
    bad = np.argwhere(d > 1e-10 * np.abs(Te).max())
    if len(bad):
        print("  bad rows", np.unique(bad[:, 0])[:40], "bad cols", np.unique(bad[:, 1])[:40])
