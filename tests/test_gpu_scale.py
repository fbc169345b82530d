"""GPU path at BASELINE.json's full sizes, in the launch configuration bench.py times.

The oracle cannot run at these sizes, so the checks are properties that hold at any size
(SURVEY 8(c) P10/P11): the known min-norm solution x0 of the seeded Gp problem (b = A x0 +
r_perp with A^T r_perp = 0), the exact rank, the normal-equation residual, the residual
identity ||A x - b|| = ||C[r:m]||, and -- sampled -- individual entries of T = U^T A V
recomputed one by one from A, V and the explicit U of a smaller run.
"""
import numpy as np
import pytest
import torch

import utv_inputs as gen

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def utv():
    from paper_2408_05238_b200 import build
    build.build()
    import paper_2408_05238_b200 as m
    return m


def _known_solution_case(utv, m, n, r, b, q, k, seed=gen.MATRIX_SEED):
    dev = torch.device("cuda:0")
    At, Bm, X0 = gen.gp_torch(m, n, r, seed=seed, device=dev, k=k)
    A0 = At.t()
    B0 = utv.colmajor(Bm)
    A = utv.colmajor(A0.clone())
    B = B0.clone()
    X, rank = utv.lstsq(A, B, utv.Opts(block=b, power_iters=q, tau=1e-10, seed=gen.SKETCH_SEED))
    torch.cuda.synchronize()
    rel = ((X - X0).norm() / X0.norm()).item()
    # normal equations ||A^T (A x - b)|| / (||A||^2 ||x||)  (A^T r_perp = 0 by construction)
    R = A0 @ X - B0
    ne = ((A0.t() @ R).norm() / (A0.norm() ** 2 * X.norm())).item()
    return rank, rel, ne


def test_cfg2_full_size(utv):
    """configs[1]: square n=20000 rank 10000, b=256, q=2, 1 RHS."""
    rank, rel, ne = _known_solution_case(utv, 20000, 20000, 10000, 256, 2, 1)
    assert rank == 10000
    assert rel <= 1e-10, rel
    assert ne <= 1e-12, ne


def test_cfg3_full_size(utv):
    """configs[2]: square n=50000 rank 25000, b=256, q=2 -- the bench workload at N=1."""
    rank, rel, ne = _known_solution_case(utv, 50000, 50000, 25000, 256, 2, 1)
    assert rank == 25000
    assert rel <= 1e-10, rel
    assert ne <= 1e-12, ne


def test_cfg4_full_size(utv):
    """configs[3]: tall m=200000 x n=20000 rank 15000, 16 RHS, q=1 (overdetermined, inconsistent)."""
    rank, rel, ne = _known_solution_case(utv, 200000, 20000, 15000, 256, 1, 16)
    assert rank == 15000
    assert rel <= 1e-10, rel
    assert ne <= 1e-12, ne


def test_residual_identity_and_sampled_T(utv):
    """P11 at a mid size: ||A x - b|| == ||C[r:m]||; sampled T_ij == (U^T A V)_ij one by one."""
    m, n, r, b = 3000, 2500, 1200, 256
    h = utv.Handle(0)
    dev = torch.device("cuda:0")
    At, Bm, _ = gen.gp_torch(m, n, r, seed=5, device=dev, k=3)
    A0 = At.t()
    A = utv.colmajor(A0.clone())
    B = utv.colmajor(Bm)
    B0 = B.clone()
    V = utv.colmajor_empty(n, n)
    U = utv.colmajor_empty(m, m)
    rank = h.factor(A, V=V, U=U, B=B, opts=utv.Opts(block=b, power_iters=2, seed=3, flags=utv.UTV_WANT_U))
    X = utv.colmajor_empty(n, 3)
    h.solve(A, V, B, rank, X)
    torch.cuda.synchronize()
    assert rank == r
    res = (A0 @ X - B0).norm().item()
    assert res == pytest.approx(B[rank:].norm().item(), rel=1e-12)
    rng = np.random.default_rng(0)
    for _ in range(64):
        i, j = int(rng.integers(0, m)), int(rng.integers(0, n))
        tij = float(U[:, i] @ (A0 @ V[:, j]))
        assert abs(float(A[i, j]) - tij) <= 1e-12 * A0.norm().item()


def test_cfg2_streamed_out_of_core(utv, monkeypatch):
    """configs[1] through the out-of-core mode (UTV_HOST_STREAMED): A in pinned host memory, only
    8192 of the 20000 columns resident in HBM; known min-norm solution and exact rank."""
    monkeypatch.setenv("UTV_OOC_MAX_RESIDENT_COLS", "8192")
    m = n = 20000
    r, b, q = 10000, 256, 2
    dev = torch.device("cuda:0")
    At, Bm, X0 = gen.gp_torch(m, n, r, seed=gen.MATRIX_SEED, device=dev, k=1)
    A0 = At.t()
    Ah = utv.colmajor_empty(m, n, device="cpu", pin_memory=True)
    Ah.copy_(A0)
    Bh = utv.colmajor(Bm).cpu()
    B0 = utv.colmajor(Bm).clone()
    Xh = utv.colmajor_empty(n, 1, device="cpu", pin_memory=True)
    h = utv.Handle(0)
    rank = h.lstsq(Ah, Bh, Xh, utv.Opts(block=b, power_iters=q, tau=1e-10, seed=gen.SKETCH_SEED,
                                          flags=utv.UTV_HOST_STREAMED))
    st = h.stream_stats()
    X = Xh.to(dev)
    rel = ((X - X0).norm() / X0.norm()).item()
    R = A0 @ X - B0
    ne = ((A0.t() @ R).norm() / (A0.norm() ** 2 * X.norm())).item()
    assert rank == r
    assert rel <= 1e-10, rel
    assert ne <= 1e-12, ne
    assert st["resident_cols"] == n - (n - 8192 + b - 1) // b * b and st["h2d_bytes"] > 8 * m * n


def test_cfg2_keep_factors_new_rhs(utv):
    """configs[1] with UTV_KEEP_FACTORS: factor + solve for one RHS, then utv_solve_rhs for a
    second, fresh RHS of the same known-solution construction (SURVEY 8(f) #3 at full size)."""
    m = n = 20000
    r, b, q = 10000, 256, 2
    dev = torch.device("cuda:0")
    At, Bm, X0 = gen.gp_torch(m, n, r, seed=gen.MATRIX_SEED, device=dev, k=2)
    A = utv.colmajor(At.t().clone())
    del At
    B = utv.colmajor(Bm)
    h = utv.Handle(0)
    X1 = utv.colmajor_empty(n, 1)
    opts = utv.Opts(block=b, power_iters=q, tau=1e-10, seed=gen.SKETCH_SEED, flags=utv.UTV_KEEP_FACTORS)
    assert h.lstsq(A, utv.colmajor(B[:, :1].clone()), X1, opts) == r
    X2 = utv.colmajor_empty(n, 1)
    assert h.solve_rhs(A, utv.colmajor(B[:, 1:2].clone()), X2) == r
    torch.cuda.synchronize()
    for j, X in ((0, X1), (1, X2)):
        rel = ((X[:, 0] - X0[:, j]).norm() / X0[:, j].norm()).item()
        assert rel <= 1e-10, (j, rel)
    h.close()


def test_cfg2_reconstruction_explicit_u(utv):
    """configs[1] with the explicit U (UTV_WANT_U, v21t): ||A - U T V^T||_F / ||A||_F and the
    orthogonality of U and V at full size (products in torch on the GPU)."""
    m = n = 20000
    r, b, q = 10000, 256, 2
    dev = torch.device("cuda:0")
    At, _, _ = gen.gp_torch(m, n, r, seed=gen.MATRIX_SEED, device=dev, k=1)
    A0 = utv.colmajor(At.t().clone())
    del At
    A = A0.clone()
    V = utv.colmajor_empty(n, n)
    U = utv.colmajor_empty(m, m)
    h = utv.Handle(0)
    rank = h.factor(A, V=V, U=U, opts=utv.Opts(block=b, power_iters=q, tau=1e-10, seed=gen.SKETCH_SEED,
                                                flags=utv.UTV_WANT_U))
    torch.cuda.synchronize()
    h.close()
    assert rank == r
    rec = ((A0 - (U @ A) @ V.t()).norm() / A0.norm()).item()
    assert rec <= 1e-13, rec
    I = torch.eye(n, dtype=torch.float64, device=dev)
    for Q in (U, V):
        E = Q.t() @ Q - I
        assert E.abs().max().item() <= 1e-13
        assert (E.norm() / n ** 0.5).item() <= 1e-13
