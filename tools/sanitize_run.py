"""Small utv_lstsq / step-level runs for compute-sanitizer (racecheck, synccheck, memcheck, initcheck).

Covers the kernels with on-chip synchronisation: the cooperative panel QR (shared-memory and
global-memory variants, grid barrier), the thread-block-cluster Jacobi SVD, the TMA/mbarrier DMMA
GEMM (every tile configuration), the block triangular solve, the wide path and the out-of-core
staging ring.  Usage: compute-sanitizer --tool racecheck python tools/sanitize_run.py [case ...]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2408_05238_b200 as utv  # noqa: E402
import utv_inputs as gen  # noqa: E402


def dev(a):
    return utv.colmajor(torch.from_numpy(np.ascontiguousarray(a)).cuda())


def check(X, X0, what, tol=1e-9):
    err = float(np.linalg.norm(X.cpu().numpy() - X0) / np.linalg.norm(X0))
    print(f"{what}: rel err vs x0 {err:.2e}", flush=True)
    assert err < tol, (what, err)


def case_lstsq():
    G = gen.GpMatrix(400, 352, 150, seed=3)
    B, X0 = G.known_rhs(k=2)
    X, r = utv.lstsq(dev(G.A), dev(B), utv.Opts(block=64, power_iters=1, tau=1e-10, seed=1))
    torch.cuda.synchronize()
    assert r == 150, r
    check(X, X0, "lstsq 400x352 b=64")


def case_lstsq_b256():
    # b = 256: the 8-CTA cluster Jacobi, 32-column sub-panels, the K = 2b fused update
    G = gen.GpMatrix(600, 560, 300, seed=4)
    B, X0 = G.known_rhs(k=1)
    X, r = utv.lstsq(dev(G.A), dev(B), utv.Opts(block=256, power_iters=1, tau=1e-10, seed=1))
    torch.cuda.synchronize()
    assert r == 300, r
    check(X, X0, "lstsq 600x560 b=256")


def case_qr_global():
    # the global-memory sub-panel variant of the cooperative panel QR
    with utv.tuned(utv.UTV_TUNE_QR_GLOBAL, 1):
        case_lstsq()


def case_gemm_cfgs():
    h = utv.default_handle()
    rng = np.random.default_rng(5)
    for cfg in range(6):
        with utv.tuned(utv.UTV_TUNE_GEMM_CFG, cfg):
            for ta, tb in ((0, 0), (1, 0), (0, 1)):
                M, N, K = 200, 72, 300
                A = rng.standard_normal((K, M) if ta else (M, K))
                Bm = rng.standard_normal((N, K) if tb else (K, N))
                Cm = np.zeros((M, N))
                Cd = dev(Cm)
                h.gemm(bool(ta), bool(tb), 1.0, dev(A), dev(Bm), 0.0, Cd)
                torch.cuda.synchronize()
                ref = (A.T if ta else A) @ (Bm.T if tb else Bm)
                e = np.abs(Cd.cpu().numpy() - ref).max() / np.abs(ref).max()
                assert e < 1e-13, (cfg, ta, tb, e)
    print("gemm cfgs 0..5 ok", flush=True)


def case_cholqr():
    """the CholeskyQR2 panel path (R22): forced on every sub-panel of a small solve (whose
    rank-transition and square panels decline, so the predicated Householder kernels run too),
    plus a tall panel with a zero column (one sub-panel accepted, one declined)"""
    with utv.tuned(utv.UTV_TUNE_QR_CHOLQR, 2):
        case_lstsq()
    h = utv.default_handle()
    rng = np.random.default_rng(8)
    P = rng.standard_normal((3000, 128))
    P[:, 70] = 0.0
    Pd, W, tau, T = h.hqr(dev(P))
    torch.cuda.synchronize()
    assert float(tau[70]) == 0.0
    Q = np.eye(3000, 128) - W.cpu().numpy() @ (T.cpu().numpy() @ W.cpu().numpy()[:128].T)
    R = np.triu(Pd.cpu().numpy())[:128]
    e = np.linalg.norm(Q @ R - P) / np.linalg.norm(P)
    assert e < 1e-13, e
    print(f"cholqr hqr 3000x128 (zero column): ||QR - P|| / ||P|| {e:.1e}", flush=True)


def case_wide():
    G = gen.GpMatrix(300, 420, 150, seed=6)
    B, X0 = G.known_rhs(k=1, consistent=True)
    X, r = utv.lstsq(dev(G.A), dev(B), utv.Opts(block=64, power_iters=1, tau=1e-10, seed=1))
    torch.cuda.synchronize()
    assert r == 150, r
    check(X, X0, "wide 300x420")


def case_ooc():
    G = gen.GpMatrix(400, 352, 150, seed=3)
    B, X0 = G.known_rhs(k=2)
    h = utv.Handle(0)
    h.set_device_budget(0)
    A = utv.colmajor(torch.from_numpy(np.ascontiguousarray(G.A)).pin_memory())
    Bh = utv.colmajor(torch.from_numpy(np.ascontiguousarray(B)).pin_memory())
    X = utv.colmajor_empty(352, 2, device="cpu", pin_memory=True)
    r = h.lstsq(A, Bh, X, utv.Opts(block=64, power_iters=1, tau=1e-10, seed=1, flags=utv.UTV_HOST_STREAMED))
    assert r == 150, r
    check(X, X0, "out-of-core 400x352")


def case_dist_ooc():
    """multi-GPU x out-of-core: an in-process group of 2 ranks streaming their host shards"""
    import threading
    from paper_2408_05238_b200 import dist as D
    os.environ["UTV_OOC_MAX_RESIDENT_COLS"] = "0"
    m, n, r, b = 400, 352, 150, 64
    G = gen.GpMatrix(m, n, r, seed=3)
    B, X0 = G.known_rhs(k=2)
    Ad = dev(G.A)
    hs = utv.local_group(2)
    shards = []
    for p in range(2):
        sh = D.scatter_columns(Ad, b, 2, p)
        t = utv.colmajor_empty(m, sh.shape[1], device="cpu", pin_memory=True)
        t.copy_(sh)
        shards.append(t)
    Bs = [dev(B) for _ in range(2)]
    Xs = [utv.colmajor_empty(n, 2) for _ in range(2)]
    out = [None, None]

    def work(p):
        out[p] = hs[p].lstsq(shards[p], Bs[p], Xs[p], utv.Opts(block=b, power_iters=1, tau=1e-10, seed=1,
                                                               flags=utv.UTV_HOST_STREAMED))
    ts = [threading.Thread(target=work, args=(p,)) for p in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    torch.cuda.synchronize()
    assert out == [150, 150], out
    check(Xs[0], X0, "dist streamed 400x352 P=2")
    for h in hs:
        h.close()


CASES = {"lstsq": case_lstsq, "lstsq256": case_lstsq_b256, "qrglobal": case_qr_global, "gemm": case_gemm_cfgs,
         "wide": case_wide, "ooc": case_ooc, "distooc": case_dist_ooc, "cholqr": case_cholqr}

if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    for nm in names:
        CASES[nm]()
    print("sanitize_run done:", " ".join(names), flush=True)
