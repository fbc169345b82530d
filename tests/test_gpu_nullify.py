"""GPU parity for Nullify_top_right_part_of_T (fig:alg_nullify_t12).

The device path zeroes T12 blockwise (n_b rows per RZ block, reading R19); the oracle sweeps
row by row.  The products of the same Householder reflectors (same dlarfg convention) give the
same T' and V' up to rounding and the sign freedom of the block SVDs, so they are compared
element by element after fixing those signs; x with nullify is the
minimum-norm solution of the rank-r approximation (pinned against pinv in the oracle tests).
"""
import numpy as np
import pytest
import torch

import oracle
import utv_inputs as gen

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


def _noisy_gd(m, n, r, tail, seed):
    rng = np.random.default_rng(seed)
    G = gen.GdMatrix(m, n, r, alpha=2.0, seed=seed)
    return G.A + tail * rng.standard_normal((m, n))


@pytest.mark.parametrize("m,n,r,b,q", [(300, 260, 100, 32, 1),    # several RZ blocks + ragged top block
                                       (200, 180, 64, 64, 0),     # r a multiple of b
                                       (150, 150, 149, 16, 1),    # nz = 1
                                       (120, 100, 7, 32, 2)])     # a single partial block
def test_factor_nullify_matches_oracle(utv, h, m, n, r, b, q):
    A = _noisy_gd(m, n, r, 1e-9, seed=50 + r)
    Ad = dev(A)
    V = dev(np.zeros((n, n)))
    rg = h.factor(Ad, V=V, opts=utv.Opts(block=b, power_iters=q, tau=1e-7, seed=6, flags=utv.UTV_NULLIFY_T12))
    T, Vg = host(Ad), host(V)
    out = oracle.randutv(A, b, q, seed=6)
    ro = oracle.rank(out["T"], 1e-7)
    assert rg == ro == r
    To, Vo = oracle.nullify(out["T"], out["V"], ro)
    # structure: T12 exactly zero, T11 upper triangular
    assert np.all(T[:r, r:] == 0.0)
    assert np.all(np.tril(T[:r, :r], -1) == 0.0)
    assert np.abs(Vg.T @ Vg - np.eye(n)).max() <= 1e-13
    # element by element against the oracle, up to the sign freedom of the block SVDs: the device
    # Jacobi sweeps pairs in a different (parallel) order than the oracle's cyclic one (DESIGN.md
    # R9), so a singular pair (u_i, v_i) may come out negated; T11' and V'(:, 0:r) are then
    # S T11'_o S and V'_o S with S = diag(+-1) (the RQ factor of U_1^T A is unique given U_1).
    S = np.sign(np.einsum("ij,ij->j", Vg[:, :r], Vo[:, :r]))
    assert np.all(S != 0)
    nA = np.linalg.norm(A)
    assert np.abs(S[:, None] * T[:r, :r] * S[None, :] - To[:r, :r]).max() <= 1e-11 * nA
    assert np.abs(Vg[:, :r] * S[None, :] - Vo[:, :r]).max() <= 1e-9


@pytest.mark.parametrize("explicit", [False, True])
@pytest.mark.parametrize("m,n,r,b,q,k", [(300, 260, 100, 32, 1, 2), (257, 200, 90, 64, 0, 1),
                                         (400, 330, 300, 128, 1, 3)])
def test_lstsq_nullify_matches_oracle(utv, m, n, r, b, q, k, explicit):
    A = _noisy_gd(m, n, r, 1e-9, seed=70 + r)
    B = np.random.default_rng(8).standard_normal((m, k))
    flags = utv.UTV_NULLIFY_T12 | (utv.UTV_EXPLICIT_V if explicit else 0)
    X, rg = utv.lstsq(dev(A), dev(B), utv.Opts(block=b, power_iters=q, tau=1e-7, seed=9, flags=flags))
    Xo, ro = oracle.lstsq(A, B, b=b, q=q, tau=1e-7, seed=9, nullify=True)
    assert rg == ro == r
    assert np.linalg.norm(host(X) - Xo) <= 1e-9 * np.linalg.norm(Xo)
    # nullify gives the smaller-norm solution than the fast option
    Xs, _ = oracle.lstsq(A, B, b=b, q=q, tau=1e-7, seed=9)
    assert np.linalg.norm(host(X)) <= np.linalg.norm(Xs) * (1 + 1e-10)


def test_lstsq_nullify_full_rank_is_noop(utv):
    """r = n: T12 is empty, so the nullify flag changes nothing."""
    G = gen.GpMatrix(200, 150, 150, seed=12)
    B, _ = G.known_rhs(k=1, consistent=True)
    X1, r1 = utv.lstsq(dev(G.A), dev(B), utv.Opts(block=32, power_iters=1, seed=2))
    X2, r2 = utv.lstsq(dev(G.A), dev(B), utv.Opts(block=32, power_iters=1, seed=2, flags=utv.UTV_NULLIFY_T12))
    assert r1 == r2 == 150
    assert np.array_equal(host(X1), host(X2))


def test_lstsq_nullify_exact_rank_equals_fast_option(utv):
    """Exact rank with a clear gap: both options give the same x (the LS solution is unique in the
    range of the row space to rounding; both are V(:,1:r) z with the same z direction)."""
    G = gen.GpMatrix(300, 240, 120, seed=13)
    B, _ = G.known_rhs(k=2)
    Xs, rs = utv.lstsq(dev(G.A), dev(B), utv.Opts(block=32, power_iters=1, seed=3))
    Xn, rn = utv.lstsq(dev(G.A), dev(B), utv.Opts(block=32, power_iters=1, seed=3, flags=utv.UTV_NULLIFY_T12))
    assert rs == rn == 120
    assert np.linalg.norm(host(Xs) - host(Xn)) <= 1e-10 * np.linalg.norm(host(Xs))


def test_lstsq_nullify_cholqr_forced(utv):
    """Nullify's blocked RZ panels (R19) and the factorization with CholeskyQR2 forced (R22)."""
    with utv.tuned(utv.UTV_TUNE_QR_CHOLQR, 2):
        test_lstsq_nullify_matches_oracle(utv, 400, 330, 300, 128, 1, 3, False)
