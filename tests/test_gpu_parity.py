"""GPU parity: the sm_100a path (through the C ABI) against the CPU oracle, element by element.

Gates: integers bit-exact (Philox words, rank r); x within 1e-9 relative
(north star, exact-rank inputs with a clear gap); step outputs within tolerances derived from
FP64 rounding (each stated in the test).  Every input is seeded and synthetic (utv_inputs).
"""
import numpy as np
import pytest
import torch

import oracle
import utv_inputs as gen

pytestmark = pytest.mark.gpu
EPS = np.finfo(np.float64).eps


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
    """numpy (any order) -> column-major float64 CUDA tensor."""
    a = np.asarray(a, dtype=np.float64)
    if a.ndim == 1:
        a = a.reshape(-1, 1)
    return torch.from_numpy(np.ascontiguousarray(a.T)).cuda().t()


def host(t):
    return t.detach().cpu().numpy()


# ----------------------------------------------------------------------------- a1
def test_philox_words_bit_exact(h):
    rng = np.random.default_rng(0)
    n = 4096
    ctr = rng.integers(0, 2**32, size=(n, 4), dtype=np.uint64).astype(np.uint32)
    key = rng.integers(0, 2**32, size=(n, 2), dtype=np.uint64).astype(np.uint32)
    ctr[0] = 0; key[0] = 0
    ctr[1] = 0xFFFFFFFF; key[1] = 0xFFFFFFFF
    out = h.philox(torch.from_numpy(ctr.view(np.int32).ravel()).cuda(), torch.from_numpy(key.view(np.int32).ravel()).cuda())
    got = host(out).view(np.uint32).reshape(n, 4)
    for i in range(0, n, 97):
        assert got[i].tolist() == oracle.philox4x32_10(ctr[i], key[i]).tolist()
    assert got[0].tolist() == [0x6627e8d5, 0xe169c58d, 0xbc57ac4c, 0x9b00dbd8]


@pytest.mark.parametrize("seed,step,row0,mrows,b", [(1, 0, 0, 1000, 64), (20240809, 7, 1234, 333, 5),
                                                     (2**40 + 3, 3, 10**6, 257, 256)])
def test_sketch_matches_oracle(h, seed, step, row0, mrows, b):
    G = host(h.sketch(seed, step, row0, mrows, b))
    Go = oracle.gauss(seed, step, row0, mrows, b)
    # libm vs CUDA log/sin/cos of the same arguments: a few ulp of max(|z|, 1)
    assert np.all(np.abs(G - Go) <= 8 * EPS * np.maximum(np.abs(Go), 1.0))


# ----------------------------------------------------------------------------- GEMM primitive
@pytest.mark.parametrize("ta,tb", [(False, False), (True, False), (False, True), (True, True)])
@pytest.mark.parametrize("M,N,K", [(1, 1, 1), (130, 67, 33), (257, 129, 300), (64, 256, 5000),
                                   (300, 17, 5000), (5000, 32, 300), (1000, 1, 2000)])   # N <= 32: narrow tile
def test_gemm_vs_numpy(h, ta, tb, M, N, K):
    rng = np.random.default_rng(M * N + K)
    A = rng.standard_normal((K, M) if ta else (M, K))
    B = rng.standard_normal((N, K) if tb else (K, N))
    C0 = rng.standard_normal((M, N))
    Cd = dev(C0)
    h.gemm(ta, tb, -0.5, dev(A), dev(B), 2.0, Cd)
    ref = -0.5 * ((A.T if ta else A) @ (B.T if tb else B)) + 2.0 * C0
    # FP64 accumulation error bound ~ K eps |A||B|
    bound = 4 * K * EPS * (np.abs(A.T if ta else A) @ np.abs(B.T if tb else B)) + 4 * EPS * np.abs(C0)
    assert np.all(np.abs(host(Cd) - ref) <= bound + 1e-300)


def test_gemm_odd_leading_dimensions(h):
    rng = np.random.default_rng(3)
    M, N, K = 71, 45, 129
    Ab = dev(rng.standard_normal((M + 3, K)))[1:M + 1]       # lda = M+3 (odd), offset -> 8-byte path
    Bb = dev(rng.standard_normal((K + 1, N)))[:K]
    Cd = dev(np.zeros((M, N)))
    h.gemm(False, False, 1.0, Ab, Bb, 0.0, Cd)
    assert np.allclose(host(Cd), host(Ab) @ host(Bb), rtol=1e-13, atol=1e-12)


# ----------------------------------------------------------------------------- a3 / a5
@pytest.mark.parametrize("m,w", [(40, 7), (300, 64), (1000, 40), (257, 256), (5000, 96), (129, 33)])
def test_hqr_matches_oracle(h, m, w):
    rng = np.random.default_rng(m + w)
    P = rng.standard_normal((m, w))
    Pd, W, tau, T = h.hqr(dev(P))
    Pk, tau_o, T_o = oracle.hqr(P)
    R_o = np.triu(Pk)[:w]
    W_o = np.tril(Pk, -1)[:, :w]; W_o[np.arange(w), np.arange(w)] = 1.0
    Pg = host(Pd)
    scale = np.linalg.norm(P)
    assert np.abs(np.triu(Pg)[:w] - R_o).max() <= 1e-13 * scale
    assert np.all(np.tril(Pg, -1) == 0.0)                        # R13
    assert np.abs(host(W) - W_o).max() <= 1e-12
    assert np.abs(host(tau) - tau_o).max() <= 1e-13
    assert np.abs(host(T) - T_o).max() <= 1e-12
    assert np.all(np.tril(host(T), -1) == 0.0)


def test_hqr_zero_and_rank_deficient_columns(h):
    P = np.zeros((300, 40)); rng = np.random.default_rng(1)
    P[:, 5] = rng.standard_normal(300); P[:, 6] = 2 * P[:, 5]; P[:, 20:] = rng.standard_normal((300, 20))
    Pd, W, tau, T = h.hqr(dev(P))
    Pk, tau_o, T_o = oracle.hqr(P)
    assert host(tau)[0] == 0.0 and tau_o[0] == 0.0
    Wg = host(W)
    Q = np.eye(300) - Wg @ host(T) @ Wg.T
    assert np.linalg.norm(Q[:, :40] @ np.triu(host(Pd))[:40] - P) <= 1e-13 * np.linalg.norm(P)


# ----------------------------------------------------------------------------- a7
@pytest.mark.parametrize("b", [1, 2, 3, 16, 33, 64, 200, 256])
def test_svd_small_matches_oracle(h, b):
    rng = np.random.default_rng(b)
    R = np.triu(rng.standard_normal((b, b)))
    Us, s, Vs, sweeps = h.svd_small(dev(R))
    _, s_o, _, _ = oracle.svd_small(R)
    s_ref = np.linalg.svd(R, compute_uv=False)
    Usg, sg, Vsg = host(Us), host(s).ravel(), host(Vs)
    assert np.abs(sg - s_o).max() <= 1e-13 * s_o[0]
    assert np.abs(sg - s_ref).max() <= 1e-13 * s_ref[0]
    # the stopping rule leaves |w_i^T w_j| <= sqrt(b) eps ||w_i|| ||w_j|| per pair, so the
    # off-diagonal of R' is bounded by ~ b eps ||R||_F (the oracle itself reaches 4.4e-14 at b = 200)
    assert np.linalg.norm(R - Usg @ np.diag(sg) @ Vsg.T) <= 4 * b * EPS * np.linalg.norm(R)
    assert np.abs(Usg.T @ Usg - np.eye(b)).max() <= 4 * b * EPS
    assert np.abs(Vsg.T @ Vsg - np.eye(b)).max() <= 1e-14
    assert 1 <= sweeps <= 30


def test_svd_small_rank_deficient(h):
    rng = np.random.default_rng(5)
    b = 64
    R = np.triu(rng.standard_normal((b, b)))
    R[:, 3] = 0.0; R[7, :] = 0.0; R[:, 40:] = 0.0
    Us, s, Vs, _ = h.svd_small(dev(R))
    s_ref = np.linalg.svd(R, compute_uv=False)
    assert np.abs(host(s).ravel() - s_ref).max() <= 1e-13 * s_ref[0]
    assert np.abs(host(Vs).T @ host(Vs) - np.eye(b)).max() <= 1e-14
    assert np.linalg.norm(R - host(Us) @ np.diag(host(s).ravel()) @ host(Vs).T) <= 1e-13 * np.linalg.norm(R)


# ----------------------------------------------------------------------------- full path
def _lstsq_gpu(utv, A, B, b, q, tau=1e-10, seed=1):
    Ad, Bd = dev(A), dev(B)
    X, r = utv.lstsq(Ad, Bd, utv.Opts(block=b, power_iters=q, tau=tau, seed=seed))
    return host(X), r


def test_cfg1_parity(utv):
    """configs[0]: square m=n=512 rank 256, b=64, q=1, single RHS -- x to 1e-9, r identical."""
    G = gen.GpMatrix(512, 512, 256)
    B, X0 = G.known_rhs(k=1)
    Xo, ro = oracle.lstsq(G.A, B, b=64, q=1, tau=1e-10, seed=gen.SKETCH_SEED)
    Xg, rg = _lstsq_gpu(utv, G.A, B, 64, 1, seed=gen.SKETCH_SEED)
    assert rg == ro == 256
    assert np.linalg.norm(Xg - Xo) <= 1e-9 * np.linalg.norm(Xo)
    assert np.linalg.norm(Xg - X0) <= 1e-10 * np.linalg.norm(X0)


@pytest.mark.parametrize("matrix", ["gp", "gd3"])
@pytest.mark.parametrize("scenario", ["ones", "perturbed"])
def test_cfg1_rhs_scenarios(utv, matrix, scenario):
    """configs[0] with the paper's right-hand-side scenarios 2 (b = ones) and
    4 (b = A x with 10% of the entries scaled by 0.999) on Gp and Gd(alpha=3)
    (SURVEY 8(d) cfg1): x to 1e-9 of the oracle, r identical, and x = the minimum-norm solution."""
    M = gen.GpMatrix(512, 512, 256) if matrix == "gp" else gen.GdMatrix(512, 512, 256, alpha=3.0)
    A = M.A
    B = gen.rhs_ones(512, 1) if scenario == "ones" else gen.rhs_perturbed(A, 1)
    Xo, ro = oracle.lstsq(A, B, b=64, q=1, tau=1e-10, seed=gen.SKETCH_SEED)
    Xg, rg = _lstsq_gpu(utv, A, B, 64, 1, seed=gen.SKETCH_SEED)
    assert rg == ro == 256
    assert np.linalg.norm(Xg - Xo) <= 1e-9 * np.linalg.norm(Xo)
    Xp = np.linalg.pinv(A, rcond=1e-10) @ B
    assert np.linalg.norm(Xg - Xp) <= 1e-9 * np.linalg.norm(Xp)


@pytest.mark.parametrize("m,n,r,b,q,kind", [
    (300, 300, 150, 64, 1, "gp"), (333, 257, 100, 64, 2, "gp"), (400, 300, 170, 32, 2, "gd"),
    (256, 256, 256, 64, 0, "full"), (200, 130, 64, 3, 1, "gd"), (600, 520, 261, 256, 1, "gp"),
    (517, 517, 200, 128, 2, "gp"), (90, 90, 0, 16, 1, "zero"), (1024, 700, 350, 256, 2, "gp"),
])
def test_lstsq_parity_sweep(utv, m, n, r, b, q, kind):
    if kind == "gp":
        M = gen.GpMatrix(m, n, r, seed=m + n)
        B, _ = M.known_rhs(k=2, consistent=m < 2 * r)
        A = M.A
    elif kind == "gd":
        M = gen.GdMatrix(m, n, r, alpha=3.0, seed=m + n)
        B, _ = M.known_rhs(k=2)
        A = M.A
    elif kind == "full":
        rng = np.random.default_rng(7)
        A = rng.standard_normal((m, n)) + n * np.eye(m, n)
        B = rng.standard_normal((m, 2))
    else:
        A = np.zeros((m, n)); B = np.ones((m, 2))
    Xo, ro = oracle.lstsq(A, B, b=b, q=q, tau=1e-10, seed=3)
    Xg, rg = _lstsq_gpu(utv, A, B, b, q, seed=3)
    assert rg == ro
    if ro == 0:
        assert np.all(Xg == 0.0)
    else:
        assert np.linalg.norm(Xg - Xo) <= 1e-9 * np.linalg.norm(Xo)


def test_factor_invariants_and_diag_parity(utv, h):
    m, n, b, q = 600, 500, 64, 1
    M = gen.GpMatrix(m, n, 230, seed=9)
    A = M.A
    B, _ = M.known_rhs(k=3)
    Ad, Bd = dev(A), dev(B)
    V = dev(np.zeros((n, n))); U = dev(np.zeros((m, m)))
    r = h.factor(Ad, V=V, U=U, B=Bd, opts=utv.Opts(block=b, power_iters=q, tau=1e-10, seed=5, flags=utv.UTV_WANT_U))
    T, Vg, Ug, Cg = host(Ad), host(V), host(U), host(Bd)
    out = oracle.randutv(A, b, q, seed=5, B=B, want_u=True)
    ro = oracle.rank(out["T"], 1e-10)
    assert r == ro == 230
    assert np.linalg.norm(A - Ug @ T @ Vg.T) <= 1e-13 * np.linalg.norm(A)
    for Q in (Ug, Vg):
        E = Q.T @ Q - np.eye(Q.shape[0])
        assert np.abs(E).max() <= 1e-13
    assert np.all(np.tril(T, -1) == 0.0)
    # every b x b diagonal block is exactly diag(sigma) (A11 := Sigma): the a9 solve of
    # the default path divides by diag(T) block by block instead of solving triangles
    for j0 in range(0, n, b):
        bw = min(b, n - j0)
        D = T[j0:j0 + bw, j0:j0 + bw]
        assert np.all(D == np.diag(np.diag(D)))
    assert np.abs(np.diag(T)[:r] - np.diag(out["T"])[:r]).max() <= 1e-11 * np.diag(out["T"])[0]
    assert np.linalg.norm(Cg - Ug.T @ B) <= 1e-12 * np.linalg.norm(B)
    X = dev(np.zeros((n, 3)))
    h.solve(Ad, V, Bd, r, X)
    Xo = oracle.solve(out["T"], out["V"], out["C"], ro)
    assert np.linalg.norm(host(X) - Xo) <= 1e-9 * np.linalg.norm(Xo)


def test_rsvd_identity_on_gpu(utv, h):
    """Remark P:848-858 with the device sketch: U(:,1:b) T(1:b,1:b) V(:,1:b)^T = A P_Y."""
    m, n, b, q, seed = 300, 240, 32, 1, 11
    A = gen.gd(m, n, 150, alpha=2.0, seed=4)
    Ad = dev(A); V = dev(np.zeros((n, n))); U = dev(np.zeros((m, m)))
    h.factor(Ad, V=V, U=U, opts=utv.Opts(block=b, power_iters=q, seed=seed, flags=utv.UTV_WANT_U))
    G = host(h.sketch(seed, 0, 0, m, b))
    Y = A.T @ G
    for _ in range(q):
        Y = A.T @ (A @ Y)
    Qy, _ = np.linalg.qr(Y)
    approx = host(U)[:, :b] @ host(Ad)[:b, :b] @ host(V)[:, :b].T
    ref = A @ Qy @ Qy.T
    assert np.linalg.norm(approx - ref) <= 1e-13 * np.linalg.norm(ref)


def test_scale_equivariance_bit_identical(utv):
    M = gen.GpMatrix(300, 260, 120, seed=13)
    B, _ = M.known_rhs(k=1)
    X1, r1 = _lstsq_gpu(utv, M.A, B, 64, 1, seed=2)
    X2, r2 = _lstsq_gpu(utv, M.A * 2.0 ** 37, B * 2.0 ** 37, 64, 1, seed=2)
    assert r1 == r2 and np.array_equal(X1, X2)


def test_deterministic_reruns(utv):
    M = gen.GpMatrix(700, 600, 300, seed=14)
    B, _ = M.known_rhs(k=1)
    X1, _ = _lstsq_gpu(utv, M.A, B, 128, 2, seed=2)
    X2, _ = _lstsq_gpu(utv, M.A, B, 128, 2, seed=2)
    assert np.array_equal(X1, X2)


def test_host_buffers_end_to_end(utv):
    M = gen.GpMatrix(400, 300, 140, seed=15)
    B, X0 = M.known_rhs(k=2)
    A_h = torch.from_numpy(M.A.T.copy()).t()            # column-major host tensors (own copies)
    B_h = torch.from_numpy(B.T.copy()).t()
    A_keep, B_keep = A_h.clone(), B_h.clone()
    X_h = torch.zeros((2, 300), dtype=torch.float64).t()
    h = utv.default_handle()
    r = h.lstsq(A_h, B_h, X_h, utv.Opts(block=64, power_iters=1, seed=1))
    assert torch.equal(A_h, A_keep) and torch.equal(B_h, B_keep)      # host inputs left unchanged
    Xo, ro = oracle.lstsq(M.A, B, b=64, q=1, seed=1)
    assert r == ro == 140
    assert np.linalg.norm(X_h.numpy() - Xo) <= 1e-9 * np.linalg.norm(Xo)


def test_error_statuses(utv, h):
    with pytest.raises(utv.UtvError) as e:                 # wide: utv_factor keeps m >= n (R4, R21)
        h.factor(dev(np.ones((3, 5))))
    assert e.value.status == utv.UTV_ERR_SHAPE
    with pytest.raises(utv.UtvError) as e:
        utv.lstsq(dev(np.ones((5, 3))), dev(np.ones((5, 1))), utv.Opts(block=0))
    assert e.value.status == utv.UTV_ERR_ARG
    with pytest.raises(utv.UtvError) as e:
        utv.lstsq(dev(np.ones((5, 3))), dev(np.ones((5, 1))), utv.Opts(block=512))
    assert e.value.status == utv.UTV_ERR_UNSUPPORTED
    A = np.ones((50, 40)); A[3, 7] = np.nan
    with pytest.raises(utv.UtvError) as e:
        utv.lstsq(dev(A), dev(np.ones((50, 1))), utv.Opts(block=16))
    assert e.value.status == utv.UTV_ERR_NUMERICAL


@pytest.mark.parametrize("m,n,r,b,q", [(600, 520, 261, 128, 2), (300, 300, 300, 64, 1), (257, 200, 90, 32, 0)])
def test_factored_v_equals_explicit_v(utv, m, n, r, b, q):
    """V = Q_1..Q_s blockdiag(V_s) applied in factored form gives the same x."""
    M = gen.GpMatrix(m, n, r, seed=31 + m)
    B, _ = M.known_rhs(k=2, consistent=m < 2 * r)
    Xf, rf = _lstsq_gpu(utv, M.A, B, b, q, seed=4)
    Ad, Bd = dev(M.A), dev(B)
    Xe, re = utv.lstsq(Ad, Bd, utv.Opts(block=b, power_iters=q, tau=1e-10, seed=4, flags=utv.UTV_EXPLICIT_V))
    Xe = host(Xe)
    assert rf == re
    assert np.linalg.norm(Xf - Xe) <= 1e-12 * np.linalg.norm(Xe)


# ----------------------------------------------------------------------------- randomized sweep
def _random_cases(count=16, seed=20241017):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(count):
        n = int(rng.integers(40, 700))
        m = n + int(rng.integers(0, 400))
        b = int(rng.choice([8, 16, 32, 48, 64, 100, 128, 256]))
        r = int(rng.integers(1, n + 1))
        out.append((m, n, r, b, int(rng.integers(0, 3)), int(rng.integers(1, 5))))
    return out


@pytest.mark.parametrize("m,n,r,b,q,k", _random_cases())
def test_lstsq_random_shapes(utv, m, n, r, b, q, k):
    """Seeded random shapes (b not dividing n, tall, rank inside a block, several RHS): r identical,
    x within 1e-9 of the oracle."""
    M = gen.GpMatrix(m, n, r, seed=m * 7 + n)
    B, _ = M.known_rhs(k=k, consistent=m < 2 * r)
    Xo, ro = oracle.lstsq(M.A, B, b=b, q=q, tau=1e-10, seed=13)
    Xg, rg = _lstsq_gpu(utv, M.A, B, b, q, seed=13)
    assert rg == ro
    assert np.linalg.norm(Xg - Xo) <= 1e-9 * max(np.linalg.norm(Xo), 1e-300)


@pytest.mark.parametrize("n,k", [(1, 1), (31, 5), (33, 16), (256, 17), (257, 40), (700, 3)])
def test_trsm_upper_blocks(utv, h, n, k):
    """a9's block back substitution (utv_trsm_upper): 32-row sub-blocks, ragged tails and RHS
    chunks of 16, against scipy's triangular solve (a library routine, not the oracle)."""
    from scipy.linalg import solve_triangular
    rng = np.random.default_rng(n * 100 + k)
    T = np.triu(rng.standard_normal((n + 3, n + 3))) / np.sqrt(n + 3) + 2.0 * np.eye(n + 3)   # ld > n
    Z = rng.standard_normal((n, k))
    ref = solve_triangular(T[:n, :n], Z, lower=False)
    Td = dev(T)
    Zd = dev(Z)
    h.trsm_upper(Td, Zd)
    torch.cuda.synchronize()
    got = Zd.cpu().numpy()
    assert np.linalg.norm(got - ref) <= 1e-13 * np.linalg.norm(ref)


def test_run_to_run_bitwise_determinism(utv):
    """Every reduction in libutv has a fixed order (split-K partials, the panel kernel's cross-CTA
    sums, the Jacobi pair schedule), so repeating a call reproduces X and T bit for bit
    (SURVEY T4); the side-stream SVD overlap does not change any arithmetic."""
    M = gen.GpMatrix(1500, 1300, 700, seed=21)
    B, _ = M.known_rhs(k=3)
    outs = []
    for _ in range(2):
        A = dev(M.A)
        Bd = dev(B)
        X = utv.colmajor_empty(1300, 3)
        r = utv.default_handle().lstsq(A, Bd, X, utv.Opts(block=256, power_iters=2, tau=1e-10, seed=8))
        torch.cuda.synchronize()
        outs.append((r, X.cpu().numpy(), A.cpu().numpy(), Bd.cpu().numpy()))
    assert outs[0][0] == outs[1][0] == 700
    for a, b in zip(outs[0][1:], outs[1][1:]):
        assert np.array_equal(a, b)
