"""Reusing one factorization for new right-hand sides.

The paper builds U explicitly in v21t because v23t, which applies U^T to B on the
fly, "cannot be later reused to solve other linear systems with a different matrix B"
(P:1726-1728).  Two device routes are checked against the oracle solving each (A, B) from scratch:
  * UTV_KEEP_FACTORS + utv_solve_rhs: U and V kept in factored form on the handle (the B200 route:
    no m x m U, about m n + n^2 / 2 doubles), single GPU and in-process multi-GPU groups;
  * UTV_WANT_U: the explicit U of v21t, C = U^T B with the library GEMM, then utv_solve.
Gates as everywhere: r identical, x within 1e-9 of the oracle.
"""
import threading

import numpy as np
import pytest
import torch

import oracle
import utv_inputs as gen
from paper_2408_05238_b200 import dist as D

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def utv():
    from paper_2408_05238_b200 import build
    build.build()
    import paper_2408_05238_b200 as m
    return m


@pytest.fixture(scope="module")
def h(utv):
    hd = utv.Handle(0)
    yield hd
    hd.close()


def dev(a):
    a = np.asarray(a, dtype=np.float64)
    if a.ndim == 1:
        a = a.reshape(-1, 1)
    return torch.from_numpy(np.ascontiguousarray(a.T)).cuda().t()


def host(t):
    return t.detach().cpu().numpy()


@pytest.mark.parametrize("m,n,r,b,q,k,explicit", [
    (600, 600, 300, 64, 1, 2, False),
    (900, 700, 333, 128, 2, 3, False),     # r inside a block, ragged last block
    (1024, 1024, 512, 256, 2, 1, True),    # UTV_EXPLICIT_V: factored V kept as well
])
def test_lstsq_keep_then_new_rhs(utv, h, m, n, r, b, q, k, explicit):
    M = gen.GpMatrix(m, n, r, seed=m + n + b)
    B1, _ = M.known_rhs(k=k, seed=1)
    flags = utv.UTV_KEEP_FACTORS | (utv.UTV_EXPLICIT_V if explicit else 0)
    opts = utv.Opts(block=b, power_iters=q, tau=1e-10, seed=7, flags=flags)
    Ad = dev(M.A)
    X1 = utv.colmajor_empty(n, k)
    r1 = h.lstsq(Ad, dev(B1), X1, opts)
    Xo, ro = oracle.lstsq(M.A, B1, b=b, q=q, tau=1e-10, seed=7)
    assert r1 == ro == r
    assert np.linalg.norm(host(X1) - Xo) <= 1e-9 * np.linalg.norm(Xo)
    for seed, kk in ((2, 1), (3, 4)):                       # two fresh right-hand sides
        B2, X02 = M.known_rhs(k=kk, seed=seed)
        Bd = dev(B2)
        X2 = utv.colmajor_empty(n, kk)
        r2 = h.solve_rhs(Ad, Bd, X2)
        Xo2, ro2 = oracle.lstsq(M.A, B2, b=b, q=q, tau=1e-10, seed=7)
        assert r2 == ro2 == r
        assert np.linalg.norm(host(X2) - Xo2) <= 1e-9 * np.linalg.norm(Xo2)
        assert np.linalg.norm(host(X2) - X02) <= 1e-10 * np.linalg.norm(X02)


def test_factor_keep_matches_explicit_factors(utv, h):
    """utv_factor with UTV_KEEP_FACTORS and explicit U, V: U^T B from the kept factors equals the
    explicit U^T B, and utv_solve_rhs equals utv_solve with the explicit V (and the oracle)."""
    m, n, r, b, q = 700, 500, 230, 64, 1
    M = gen.GpMatrix(m, n, r, seed=19)
    A = M.A
    Ad = dev(A)
    V = utv.colmajor_empty(n, n); U = utv.colmajor_empty(m, m)
    rk = h.factor(Ad, V=V, U=U, opts=utv.Opts(block=b, power_iters=q, tau=1e-10, seed=5,
                                               flags=utv.UTV_WANT_U | utv.UTV_KEEP_FACTORS))
    assert rk == r
    B2, X02 = M.known_rhs(k=3, seed=11)
    Bd = dev(B2)
    X = utv.colmajor_empty(n, 3)
    assert h.solve_rhs(Ad, Bd, X) == r
    Ug = host(U)
    assert np.linalg.norm(host(Bd) - Ug.T @ B2) <= 1e-12 * np.linalg.norm(B2)      # kept U^T B
    X_explicit = utv.colmajor_empty(n, 3)
    h.solve(Ad, V, dev(Ug.T @ B2), r, X_explicit)                                    # v21t route
    Xo, ro = oracle.lstsq(A, B2, b=b, q=q, tau=1e-10, seed=5)
    assert ro == r
    for Xg in (host(X), host(X_explicit)):
        assert np.linalg.norm(Xg - Xo) <= 1e-9 * np.linalg.norm(Xo)
        assert np.linalg.norm(Xg - X02) <= 1e-10 * np.linalg.norm(X02)


def test_explicit_u_route_new_rhs(utv, h):
    """v21t: factor once with the explicit U, then C = U^T B_new (library GEMM) and
    utv_solve for two fresh right-hand sides."""
    m, n, r, b, q = 800, 640, 300, 128, 2
    M = gen.GpMatrix(m, n, r, seed=23)
    Ad = dev(M.A)
    V = utv.colmajor_empty(n, n); U = utv.colmajor_empty(m, m)
    rk = h.factor(Ad, V=V, U=U, opts=utv.Opts(block=b, power_iters=q, tau=1e-10, seed=9, flags=utv.UTV_WANT_U))
    for seed in (4, 5):
        B, _ = M.known_rhs(k=2, seed=seed)
        Cd = utv.colmajor_empty(m, 2)
        h.gemm(True, False, 1.0, U, dev(B), 0.0, Cd)
        X = utv.colmajor_empty(n, 2)
        h.solve(Ad, V, Cd, rk, X)
        Xo, ro = oracle.lstsq(M.A, B, b=b, q=q, tau=1e-10, seed=9)
        assert rk == ro == r
        assert np.linalg.norm(host(X) - Xo) <= 1e-9 * np.linalg.norm(Xo)


def test_keep_errors(utv, h):
    M = gen.GpMatrix(300, 200, 100, seed=3)
    Ad = dev(M.A)
    X = utv.colmajor_empty(200, 1)
    with pytest.raises(utv.UtvError) as e:                            # UTV_NULLIFY_T12 not kept
        h.factor(Ad, opts=utv.Opts(block=64, power_iters=1, flags=utv.UTV_KEEP_FACTORS | utv.UTV_NULLIFY_T12))
    assert e.value.status == utv.UTV_ERR_UNSUPPORTED
    h2 = utv.Handle(0)
    with pytest.raises(utv.UtvError) as e:                            # nothing kept on a fresh handle
        h2.solve_rhs(Ad, dev(np.ones((300, 1))), X)
    assert e.value.status == utv.UTV_ERR_ARG
    h2.lstsq(dev(M.A), dev(np.ones((300, 1))), X, utv.Opts(block=64, power_iters=1, flags=utv.UTV_KEEP_FACTORS))
    with pytest.raises(utv.UtvError) as e:                            # m differs from the kept one
        h2.solve_rhs(Ad, dev(np.ones((301, 1))), X)
    assert e.value.status == utv.UTV_ERR_SHAPE
    with pytest.raises(utv.UtvError) as e:                            # host A
        Ah = torch.from_numpy(np.ascontiguousarray(M.A.T)).t()
        h2.lstsq(Ah, torch.ones(300, 1, dtype=torch.float64), torch.zeros(200, 1, dtype=torch.float64),
                 utv.Opts(block=64, power_iters=1, flags=utv.UTV_KEEP_FACTORS))
    assert e.value.status == utv.UTV_ERR_UNSUPPORTED
    h2.close()


@pytest.mark.parametrize("P,m,n,r,b,q", [(2, 600, 600, 300, 64, 1), (3, 700, 550, 260, 64, 2)])
def test_local_group_keep_then_new_rhs(utv, P, m, n, r, b, q):
    """Multi-GPU handles (in-process group, block-cyclic shards): every rank keeps the broadcast
    W_U / T_U / U_s and the replicated factored V; utv_solve_rhs runs the distributed triangular
    solve on the shards of T."""
    M = gen.GpMatrix(m, n, r, seed=m + n + P)
    B1, _ = M.known_rhs(k=1, seed=1)
    B2, X02 = M.known_rhs(k=2, seed=2)
    handles = utv.local_group(P)
    Ad = dev(M.A)
    shards = [utv.colmajor(D.scatter_columns(Ad, b, P, p).clone()) for p in range(P)]
    opts = utv.Opts(block=b, power_iters=q, tau=1e-10, seed=3, flags=utv.UTV_KEEP_FACTORS)
    X1 = [utv.colmajor_empty(n, 1) for _ in range(P)]
    X2 = [utv.colmajor_empty(n, 2) for _ in range(P)]
    Bs1 = [dev(B1) for _ in range(P)]
    Bs2 = [dev(B2) for _ in range(P)]
    torch.cuda.synchronize()
    out, err = [None] * P, [None] * P

    def work(p):
        try:
            handles[p].lstsq(shards[p], Bs1[p], X1[p], opts)
            out[p] = handles[p].solve_rhs(shards[p], Bs2[p], X2[p], m=m)
            handles[p].synchronize()
        except Exception as e:          # noqa: BLE001 -- re-raised below
            err[p] = e

    ts = [threading.Thread(target=work, args=(p,)) for p in range(P)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=600)
    assert not any(t.is_alive() for t in ts), "a rank hung"
    for e in err:
        if e is not None:
            raise e
    torch.cuda.synchronize()
    Xo, ro = oracle.lstsq(M.A, B2, b=b, q=q, tau=1e-10, seed=3)
    assert all(o == ro == r for o in out)
    X2h = [host(X) for X in X2]
    for Xg in X2h:
        assert np.array_equal(Xg, X2h[0])
        assert np.linalg.norm(Xg - Xo) <= 1e-9 * np.linalg.norm(Xo)
    for hd in handles:
        hd.close()


def test_keep_then_new_rhs_cholqr_forced(utv, h):
    """Factor reuse for a new right-hand side with CholeskyQR2 panels forced
    (R22): the kept W_U / T_U from the reconstruction serve later solves exactly as well."""
    with utv.tuned(utv.UTV_TUNE_QR_CHOLQR, 2):
        test_lstsq_keep_then_new_rhs(utv, h, 900, 700, 333, 128, 2, 3, False)
