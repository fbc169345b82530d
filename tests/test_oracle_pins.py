"""Pins of the CPU oracle to values fixed by the paper and by mathematics (not by itself).

Every test here runs on CPU (`-m "not gpu"`).  The pins:
P1 Philox KATs, P2 Gaussian moments, P3/P4 Householder QR + T-factor, P5 Jacobi SVD,
P6 randUTV invariants, P7 the RSVD identity, P8 rank, P9 small solves
against brute-force pinv / numpy.linalg.solve / QR-LS, P10 known solution,
P11 residual identity, P12 power-of-two scale equivariance, P13 multi-RHS.
"""
import math
import os

import numpy as np
import pytest

import oracle
import utv_inputs as gen

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
EPS = np.finfo(np.float64).eps


def _golden_examples():
    out = {}
    for line in open(os.path.join(GOLDEN, "worked_examples.txt")):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        key, *vals = line.split()
        out[key] = np.array([float(v) for v in vals])
    return out


# --------------------------------------------------------------------------- P1
def test_philox_kat():
    for line in open(os.path.join(GOLDEN, "philox_kat.txt")):
        if line.startswith("#") or not line.strip():
            continue
        w = [int(x, 16) for x in line.split() if x != "->"]
        ctr, key, want = w[0:4], w[4:6], w[6:10]
        assert oracle.philox4x32_10(ctr, key).tolist() == want


# --------------------------------------------------------------------------- P2
def test_gauss_moments_and_layout():
    G = oracle.gauss(seed=7, step=3, row0=100, mrows=50000, b=2)
    z = G.ravel()
    assert abs(z.mean()) < 0.02 and abs(z.var() - 1.0) < 0.05
    # counter layout R6: entry (i, c) depends only on (seed, step, row0 + i, c) -> a shifted
    # block of rows equals the corresponding rows of a larger block
    G1 = oracle.gauss(seed=7, step=3, row0=0, mrows=130, b=5)
    G2 = oracle.gauss(seed=7, step=3, row0=100, mrows=30, b=5)
    assert np.array_equal(G1[100:130], G2)
    # odd b drops z_odd of the last pair: the first 4 columns equal the b=4 block
    G3 = oracle.gauss(seed=7, step=3, row0=0, mrows=130, b=4)
    assert np.array_equal(G1[:, :4], G3)
    # different steps / seeds give different streams
    assert not np.array_equal(oracle.gauss(7, 4, 0, 130, 5), G1)
    assert not np.array_equal(oracle.gauss(8, 3, 0, 130, 5), G1)


def test_gauss_box_muller_closed_form():
    """Entry (i, c) equals Box-Muller of the KAT-pinned Philox words (R6)."""
    seed, step, row0 = 0x1234_5678_9ABC, 5, 17
    G = oracle.gauss(seed, step, row0, 4, 6)
    key = [seed & 0xFFFFFFFF, seed >> 32]
    for i in range(4):
        g = row0 + i
        for c in range(0, 6, 2):
            x = oracle.philox4x32_10([g & 0xFFFFFFFF, g >> 32, c // 2, step], key)
            u1 = (((int(x[0]) << 32 | int(x[1])) >> 11) + 1) * 2.0 ** -53
            u2 = (((int(x[2]) << 32 | int(x[3])) >> 11) + 1) * 2.0 ** -53
            rad = math.sqrt(-2.0 * math.log(u1))
            assert G[i, c] == pytest.approx(rad * math.cos(2 * math.pi * u2), rel=4 * EPS, abs=4 * EPS)
            assert G[i, c + 1] == pytest.approx(rad * math.sin(2 * math.pi * u2), rel=4 * EPS, abs=4 * EPS)


# --------------------------------------------------------------------------- P3 / P4
def _unpack(Pk, tau, T):
    m, n = Pk.shape
    W = np.tril(Pk, -1)[:, :n].copy()
    W[np.arange(n), np.arange(n)] = 1.0
    R = np.triu(Pk)[:n, :]
    return W, R


def test_hqr_worked_example():
    ex = _golden_examples()
    Pk, tau, T = oracle.hqr(ex["hqr_x"].reshape(2, 1))
    assert Pk[0, 0] == ex["hqr_R"][0]
    assert tau[0] == pytest.approx(ex["hqr_tau"][0], rel=2 * EPS)
    assert Pk[1, 0] == pytest.approx(ex["hqr_v"][1], rel=2 * EPS)


@pytest.mark.parametrize("m,n", [(40, 7), (64, 64), (300, 32), (33, 1)])
def test_hqr_reconstruction_and_tfactor(m, n):
    rng = np.random.default_rng(m * 100 + n)
    P = rng.standard_normal((m, n))
    Pk, tau, T = oracle.hqr(P)
    W, R = _unpack(Pk, tau, T)
    Q = np.eye(m) - W @ T @ W.T
    # P4: compact WY equals the explicit product H_0 ... H_{n-1}
    H = np.eye(m)
    for j in range(n):
        v = W[:, j]
        H = H @ (np.eye(m) - tau[j] * np.outer(v, v))
    assert np.abs(Q - H).max() <= 1e-15 * max(1, m / 8)
    # P3: Q R = P, Q orthogonal, T upper triangular
    assert np.linalg.norm(Q[:, :n] @ R - P) <= 100 * EPS * np.linalg.norm(P)
    assert np.linalg.norm(Q.T @ Q - np.eye(m)) <= 100 * EPS * max(n, 1) * math.sqrt(m / n)
    assert np.array_equal(np.tril(T, -1), np.zeros_like(T))
    # R diagonal follows dlarfg: |R_jj| = column norm of the reduced matrix; Q^T P = [R; 0]
    assert np.allclose((Q.T @ P)[n:], 0.0, atol=100 * EPS * np.linalg.norm(P))


def test_hqr_zero_column_gives_identity_reflector():
    P = np.zeros((6, 3)); P[:, 1] = np.arange(1, 7)
    Pk, tau, T = oracle.hqr(P)
    assert tau[0] == 0.0 and Pk[0, 0] == 0.0
    W, R = _unpack(Pk, tau, T)
    Q = np.eye(6) - W @ T @ W.T
    assert np.linalg.norm(Q[:, :3] @ R - P) <= 1e-14 * np.linalg.norm(P)


# --------------------------------------------------------------------------- P5
def test_svd_worked_examples():
    ex = _golden_examples()
    _, s, _, _ = oracle.svd_small(np.diag([3.0, 1.0]))
    assert np.allclose(s, ex["svd_diag31"], rtol=0, atol=1e-15)
    _, s, _, _ = oracle.svd_small(np.array([[0.0, 1.0], [1.0, 0.0]]))
    assert np.allclose(s, ex["svd_swap"], rtol=0, atol=1e-15)


@pytest.mark.parametrize("b", [1, 2, 8, 31, 64])
def test_svd_small_random(b):
    rng = np.random.default_rng(b)
    R = np.triu(rng.standard_normal((b, b)))
    Us, s, Vs, sweeps = oracle.svd_small(R)
    ref = np.linalg.svd(R, compute_uv=False)
    assert np.allclose(s, ref, rtol=1e-14, atol=1e-14 * ref[0])
    assert np.all(np.diff(s) <= 0) and np.all(s >= 0)
    assert np.linalg.norm(R - Us @ np.diag(s) @ Vs.T) <= 10 * math.sqrt(b) * EPS * np.linalg.norm(R)
    # U_s accumulates O(sweeps * b) rotations; V_s comes from a Householder QR (R9)
    assert np.abs(Us.T @ Us - np.eye(b)).max() <= 4 * b * EPS
    assert np.abs(Vs.T @ Vs - np.eye(b)).max() <= 1e-14
    assert sweeps <= 30


def test_svd_small_rank_deficient_completes_both_factors():
    rng = np.random.default_rng(5)
    b = 16
    R = np.triu(rng.standard_normal((b, b)))
    R[:, 3] = 0.0; R[7, :] = 0.0; R[:, 11] = 0.0
    Us, s, Vs, _ = oracle.svd_small(R)
    ref = np.linalg.svd(R, compute_uv=False)
    assert np.allclose(s, ref, atol=1e-14 * ref[0])
    assert np.abs(Us.T @ Us - np.eye(b)).max() <= 1e-14
    assert np.abs(Vs.T @ Vs - np.eye(b)).max() <= 1e-14
    assert np.linalg.norm(R - Us @ np.diag(s) @ Vs.T) <= 1e-14 * np.linalg.norm(R)


# --------------------------------------------------------------------------- P6 / P7
def _check_utv(A, out, b, rec_tol=1e-13):
    T, V, U = out["T"], out["V"], out["U"]
    m, n = A.shape
    rec = np.linalg.norm(A - U @ T @ V.T) / np.linalg.norm(A)
    assert rec <= rec_tol, rec
    for Q in (U, V):
        E = Q.T @ Q - np.eye(Q.shape[0])
        assert np.abs(E).max() <= 1e-13 and np.linalg.norm(E) / math.sqrt(Q.shape[0]) <= 1e-13
    assert np.array_equal(np.tril(T, -1), np.zeros_like(T))
    for j0 in range(0, n, b):
        j1 = min(n, j0 + b)
        blk = T[j0:j1, j0:j1]
        d = np.diag(blk)
        assert np.array_equal(blk, np.diag(d)), "diagonal block not diagonal"
        # non-increasing; numerically-zero columns (R9b) may reorder at the rounding level
        assert np.all(d >= 0) and np.all(np.diff(d) <= 8 * EPS * np.linalg.norm(A))


@pytest.mark.parametrize("m,n,r,b,q", [(96, 96, 48, 16, 1), (120, 80, 50, 16, 2), (11, 8, 5, 3, 1),
                                       (64, 64, 64, 64, 0), (70, 50, 50, 7, 1)])
def test_randutv_invariants(m, n, r, b, q):
    A = gen.gp(m, n, r, seed=m + n + r)
    out = oracle.randutv(A, b, q, seed=1, want_u=True)
    _check_utv(A, out, b)


def test_randutv_invariants_decay():
    A = gen.gd(100, 90, 70, alpha=3.0, seed=3)
    out = oracle.randutv(A, 16, 2, seed=2, want_u=True)
    _check_utv(A, out, 16)


def test_randutv_rsvd_identity():
    """Remark P:848-858: U(:,1:b) T(1:b,1:b) V(:,1:b)^T is exactly the RSVD rank-b approximation
    A P_Y, P_Y the projector onto span((A^T A)^q A^T G) -- G the step-0 sketch (R6)."""
    m, n, b, q, seed = 80, 60, 12, 1, 9
    A = gen.gd(m, n, 40, alpha=2.0, seed=4)
    out = oracle.randutv(A, b, q, seed=seed, want_u=True)
    G = oracle.gauss(seed, 0, 0, m, b)
    Y = A.T @ G
    for _ in range(q):
        Y = A.T @ (A @ Y)
    Qy, _ = np.linalg.qr(Y)
    approx = out["U"][:, :b] @ out["T"][:b, :b] @ out["V"][:, :b].T
    ref = A @ Qy @ Qy.T
    assert np.linalg.norm(approx - ref) <= 1e-13 * np.linalg.norm(ref)


def test_randutv_b_equal_n_is_qr_plus_svd():
    """n <= b: no sketch (R5); T = diag(singular values of A)."""
    A = np.random.default_rng(1).standard_normal((30, 10))
    out = oracle.randutv(A, 16, 1, seed=1, want_u=True)
    s = np.linalg.svd(A, compute_uv=False)
    assert np.allclose(np.diag(out["T"])[:10], s, rtol=1e-13)
    _check_utv(A, out, 16)


def test_randutv_rejects_wide_and_bad_args():
    with pytest.raises(oracle.OracleError):
        oracle.randutv(np.ones((3, 5)), 2, 1, 1)
    with pytest.raises(oracle.OracleError):
        oracle.randutv(np.ones((5, 3)), 0, 1, 1)


# --------------------------------------------------------------------------- P8 / P9
def _pinv_solution(A, B, tau):
    U, s, Vt = np.linalg.svd(A, full_matrices=False)
    keep = s > tau * s[0] if s.size and s[0] > 0 else np.zeros_like(s, bool)
    return Vt[keep].T @ ((U[:, keep].T @ B) / s[keep, None])


def test_lstsq_worked_example():
    ex = _golden_examples()
    A = ex["lstsq_A"].reshape(2, 2)
    X, r = oracle.lstsq(A, ex["lstsq_b"], b=1, q=1, tau=1e-10, seed=1)
    assert r == 1
    assert np.allclose(X.ravel(), ex["lstsq_x"], atol=1e-15)
    assert np.linalg.norm(A @ X.ravel() - ex["lstsq_b"]) == pytest.approx(ex["lstsq_res"][0], abs=1e-15)


@pytest.mark.parametrize("m,n,r,b", [(24, 24, 10, 4), (40, 30, 17, 8), (64, 64, 33, 16), (50, 20, 20, 3),
                                     (36, 36, 8, 2), (11, 8, 5, 3), (60, 45, 45, 16)])
@pytest.mark.parametrize("q", [0, 2])
def test_lstsq_matches_pinv_exact_rank(m, n, r, b, q):
    Gd = gen.GdMatrix(m, n, r, alpha=1.0, seed=m * n + r)
    B, X0 = Gd.known_rhs(k=2)
    X, rk = oracle.lstsq(Gd.A, B, b=b, q=q, tau=1e-10, seed=3)
    assert rk == r
    Xp = _pinv_solution(Gd.A, B, 1e-10)
    assert np.linalg.norm(X - Xp) <= 1e-11 * np.linalg.norm(Xp)


def test_lstsq_full_rank_square_and_tall():
    rng = np.random.default_rng(0)
    A = rng.standard_normal((60, 60)) + 60 * np.eye(60)
    bvec = rng.standard_normal(60)
    X, r = oracle.lstsq(A, bvec, b=16, q=1)
    assert r == 60
    assert np.linalg.norm(X.ravel() - np.linalg.solve(A, bvec)) <= 1e-13 * np.linalg.norm(X)
    A = rng.standard_normal((90, 40))
    bvec = rng.standard_normal(90)
    X, r = oracle.lstsq(A, bvec, b=16, q=1)
    Qa, Ra = np.linalg.qr(A)                      # A2: x = R^{-1} Q^T b
    assert r == 40
    assert np.linalg.norm(X.ravel() - np.linalg.solve(Ra, Qa.T @ bvec)) <= 1e-12 * np.linalg.norm(X)


@pytest.mark.parametrize("m,n,r,b,q", [(20, 30, 8, 4, 1), (30, 64, 30, 16, 2), (11, 40, 5, 3, 0),
                                       (33, 50, 17, 8, 2), (1, 7, 1, 4, 1), (48, 49, 20, 16, 0)])
def test_lstsq_wide_matches_pinv_exact_rank(m, n, r, b, q):
    """R21 (m < n via randUTV of A^T): the min-norm solution on exact-rank inputs (brute-force pinv)."""
    Gd = gen.GdMatrix(m, n, r, alpha=1.0, seed=m * n + r)
    B, X0 = Gd.known_rhs(k=2, consistent=r == m)
    X, rk = oracle.lstsq(Gd.A, B, b=b, q=q, tau=1e-10, seed=5)
    assert X.shape == (n, 2) and rk == r
    Xp = _pinv_solution(Gd.A, B, 1e-10)
    assert np.linalg.norm(X - Xp) <= 1e-11 * np.linalg.norm(Xp)
    assert np.linalg.norm(X - X0) <= 1e-11 * np.linalg.norm(X0)


def test_lstsq_wide_full_row_rank_closed_form():
    """Full row rank: x = A^T (A A^T)^{-1} b, the textbook minimum-norm solution."""
    rng = np.random.default_rng(7)
    A = rng.standard_normal((25, 60))
    bvec = rng.standard_normal(25)
    X, r = oracle.lstsq(A, bvec, b=8, q=1)
    assert r == 25
    xc = A.T @ np.linalg.solve(A @ A.T, bvec)
    assert np.linalg.norm(X.ravel() - xc) <= 1e-12 * np.linalg.norm(xc)
    assert np.linalg.norm(A @ X.ravel() - bvec) <= 1e-12 * np.linalg.norm(bvec)


def test_lstsq_wide_zero_and_nullify_rejected():
    X, r = oracle.lstsq(np.zeros((4, 9)), np.ones(4), b=2, q=1)
    assert r == 0 and X.shape == (9, 1) and not X.any()
    with pytest.raises(oracle.OracleError):
        oracle.lstsq(np.ones((3, 5)), np.ones(3), b=2, q=1, nullify=True)


@pytest.mark.parametrize("scenario", ["ones", "perturbed"])
def test_cfg1_rhs_scenarios_min_norm(scenario):
    """cfg1 with the paper's RHS scenarios 2 and 4: on the exact-rank
    Gp matrix the fast-option x is the minimum-norm solution (brute-force pinv)."""
    G = gen.GpMatrix(512, 512, 256)
    B = gen.rhs_ones(512, 1) if scenario == "ones" else gen.rhs_perturbed(G.A, 1)
    X, r = oracle.lstsq(G.A, B, b=64, q=1, tau=1e-10, seed=gen.SKETCH_SEED)
    assert r == 256
    Xp = _pinv_solution(G.A, B, 1e-10)
    assert np.linalg.norm(X - Xp) <= 1e-12 * np.linalg.norm(Xp)


def test_rank_edge_cases():
    X, r = oracle.lstsq(np.zeros((10, 6)), np.ones(10), b=4, q=1)
    assert r == 0 and np.all(X == 0.0)
    T = np.diag([5.0, 4.0, 1e-12, 3.0])
    assert oracle.rank(T, 1e-10) == 2                # prefix rule (R10)
    assert oracle.rank(np.diag([2.0, 1.0]), 0.0) == 2


# --------------------------------------------------------------------------- P10 / P11 / P13
def test_known_solution_gp():
    G = gen.GpMatrix(240, 240, 100, seed=11)
    B, X0 = G.known_rhs(k=1)
    X, r = oracle.lstsq(G.A, B, b=32, q=2, tau=1e-10, seed=1)
    assert r == 100
    assert np.linalg.norm(X - X0) <= 1e-10 * np.linalg.norm(X0)
    A = G.A
    assert np.linalg.norm(A.T @ (A @ X - B)) / (np.linalg.norm(A) ** 2 * np.linalg.norm(X)) <= 1e-12


def test_residual_identity_and_multi_rhs():
    G = gen.GpMatrix(200, 150, 70, seed=12)
    B, X0 = G.known_rhs(k=3)
    out = oracle.randutv(G.A, 16, 1, seed=1, B=B)
    r = oracle.rank(out["T"], 1e-10)
    X = oracle.solve(out["T"], out["V"], out["C"], r)
    res = np.linalg.norm(G.A @ X - B)
    assert res == pytest.approx(np.linalg.norm(out["C"][r:]), rel=1e-12)        # P11
    for c in range(3):                                                            # P13
        Xc, rc = oracle.lstsq(G.A, B[:, c], b=16, q=1, tau=1e-10, seed=1)
        assert rc == r
        assert np.linalg.norm(Xc.ravel() - X[:, c]) <= 1e-12 * np.linalg.norm(X[:, c])


# --------------------------------------------------------------------------- P12
def test_scale_equivariance_bit_identical():
    G = gen.GpMatrix(96, 80, 40, seed=13)
    B, _ = G.known_rhs(k=1)
    X1, r1 = oracle.lstsq(G.A, B, b=16, q=1, seed=2)
    s = 2.0 ** 37
    X2, r2 = oracle.lstsq(G.A * s, B * s, b=16, q=1, seed=2)
    assert r1 == r2 and np.array_equal(X1, X2)


def _randutv_steps(A, b, q, seed, top_rows):
    """randUTV assembled from the oracle's step functions (gauss, hqr, svd_small) with the right
    update of fig:alg_utv applied either to ALL rows 0:m (reading R1) or, literally as Fig. 2
    prints it, only to the trailing rows j0:m.  Returns (U, T, V)."""
    A = np.array(A, dtype=np.float64)
    m, n = A.shape
    U, V = np.eye(m), np.eye(n)

    def q_of(Pk, tau, T):
        W = np.tril(Pk, -1); W[np.arange(Pk.shape[1]), np.arange(Pk.shape[1])] = 1.0
        return np.eye(Pk.shape[0]) - W @ T @ W.T

    for step, j0 in enumerate(range(0, n, b)):
        bw = min(b, n - j0)
        if n - j0 > b:
            G = oracle.gauss(seed, step, j0, m - j0, b)
            Ap = A[j0:, j0:]
            Y = Ap.T @ G
            for _ in range(q):
                Y = Ap.T @ (Ap @ Y)
            Qv = np.eye(n)
            Qv[j0:, j0:] = q_of(*oracle.hqr(Y))
            r0 = 0 if top_rows else j0
            A[r0:, :] = A[r0:, :] @ Qv
            V = V @ Qv
        Pk, tau, T = oracle.hqr(A[j0:, j0:j0 + bw])
        Qu = np.eye(m)
        Qu[j0:, j0:] = q_of(Pk, tau, T)
        A = Qu.T @ A
        U = U @ Qu
        A[j0 + bw:, j0:j0 + bw] = 0.0
        Us, s, Vs, _ = oracle.svd_small(np.triu(A[j0:j0 + bw, j0:j0 + bw]))
        A[j0:j0 + bw, j0:j0 + bw] = np.diag(s)
        A[:j0, j0:j0 + bw] = A[:j0, j0:j0 + bw] @ Vs
        A[j0:j0 + bw, j0 + bw:] = Us.T @ A[j0:j0 + bw, j0 + bw:]
        V[:, j0:j0 + bw] = V[:, j0:j0 + bw] @ Vs
        U[:, j0:j0 + bw] = U[:, j0:j0 + bw] @ Us
    return U, A, V


def test_literal_fig2_reading_is_wrong():
    """R1 (P:798-801 vs P:824, Appl_r_TD): the right update printed in Fig. 2 touches
    only [A11 A12; A21 A22]; run literally (rows j0:m only) the factors no longer reproduce A,
    while the all-rows reading does.  Both runs use the oracle's own step functions."""
    A = gen.gp(64, 64, 32, seed=2)
    nrm = np.linalg.norm(A)
    U, T, V = _randutv_steps(A, 16, 1, 1, top_rows=True)
    assert np.linalg.norm(A - U @ T @ V.T) <= 1e-13 * nrm
    U, T, V = _randutv_steps(A, 16, 1, 1, top_rows=False)
    assert np.linalg.norm(A - U @ T @ V.T) >= 1e-3 * nrm          # 3e-2
    # the all-rows assembly is the C oracle's randutv (same T up to rounding)
    out = oracle.randutv(A, 16, 1, seed=1, want_u=True)
    Ua, Ta, Va = _randutv_steps(A, 16, 1, 1, top_rows=True)
    assert np.abs(out["T"] - Ta).max() <= 1e-10 * nrm


def test_threads_bit_identical():
    G = gen.GpMatrix(128, 128, 60, seed=14)
    B, _ = G.known_rhs(k=1)
    n0 = oracle.get_threads()
    try:
        oracle.set_threads(1)
        X1, _ = oracle.lstsq(G.A, B, b=16, q=1)
        oracle.set_threads(4)
        X4, _ = oracle.lstsq(G.A, B, b=16, q=1)
    finally:
        oracle.set_threads(n0)
    assert np.array_equal(X1, X4)


# --------------------------------------------------------------------------- Nullify
def _noisy_gd(m, n, r, tail, seed):
    """Gd with an exact-rank part plus a small full-rank tail (numerical rank r, no exact gap)."""
    rng = np.random.default_rng(seed)
    G = gen.GdMatrix(m, n, r, alpha=2.0, seed=seed)
    return G.A + tail * rng.standard_normal((m, n)), G


def test_nullify_structure_and_exact_rank_invariance():
    G = gen.GpMatrix(150, 120, 50, seed=41)
    A = G.A
    B, _ = G.known_rhs(k=2)
    out = oracle.randutv(A, 16, 1, seed=3, B=B, want_u=True)
    r = oracle.rank(out["T"], 1e-10)
    assert r == 50
    T2, V2 = oracle.nullify(out["T"], out["V"], r)
    assert np.all(T2[:r, r:] == 0.0)
    assert np.all(np.tril(T2[:r, :r], -1) == 0.0)
    assert np.abs(V2.T @ V2 - np.eye(120)).max() <= 1e-13
    # exact rank: T22 ~ 0, so A = U T' V'^T still holds
    assert np.linalg.norm(A - out["U"] @ T2 @ V2.T) <= 1e-13 * np.linalg.norm(A)
    Xs, rs = oracle.lstsq(A, B, b=16, q=1, seed=3)
    Xn, rn = oracle.lstsq(A, B, b=16, q=1, seed=3, nullify=True)
    assert rs == rn and np.linalg.norm(Xs - Xn) <= 1e-12 * np.linalg.norm(Xs)


@pytest.mark.parametrize("q", [0, 1])
def test_nullify_gives_min_norm_solution_of_truncated_factorization(q):
    """x_nullify = pinv(U_1 [T11 T12] V^T) b (brute force), the min-norm LS solution of the rank-r
    COD; x_simple only minimises the residual and has a larger norm."""
    m, n, r, b = 90, 70, 40, 8
    A, _ = _noisy_gd(m, n, r, 1e-8, seed=43 + q)
    rng = np.random.default_rng(5)
    B = rng.standard_normal((m, 1))
    out = oracle.randutv(A, b, q, seed=2, B=B, want_u=True)
    rk = oracle.rank(out["T"], 1e-6)
    assert rk == r
    T, V, U = out["T"], out["V"], out["U"]
    Ahat = U[:, :rk] @ T[:rk, :] @ V.T
    Xref = np.linalg.pinv(Ahat, rcond=1e-12) @ B
    Xn, rn = oracle.lstsq(A, B, b=b, q=q, tau=1e-6, seed=2, nullify=True)
    Xs, rs = oracle.lstsq(A, B, b=b, q=q, tau=1e-6, seed=2)
    assert rn == rs == r
    assert np.linalg.norm(Xn - Xref) <= 1e-9 * np.linalg.norm(Xref)
    assert np.linalg.norm(Xn) <= np.linalg.norm(Xs) * (1 + 1e-12)
    # both minimise the residual of the truncated problem
    assert np.linalg.norm(Ahat @ Xn - B) == pytest.approx(np.linalg.norm(Ahat @ Xs - B), rel=1e-10)
