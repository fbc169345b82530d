"""Native multi-GPU path (utv_create_local_group / utv_create_dist) against the oracle.

The in-process group runs P ranks as host threads on ONE GPU (each rank its own handle and
stream, collectives combined in rank order), so the block-cyclic orchestration, the collectives'
payloads and the owner logic are exercised at P = 2..5 on the single GPU this round has; the NCCL
communicator is checked at P = 1 (NCCL refuses two ranks on one device).  Gates: r identical on
every rank and equal to the oracle's, X identical on every rank and within 1e-9 of the oracle.
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


def dev(a):
    a = np.asarray(a, dtype=np.float64)
    if a.ndim == 1:
        a = a.reshape(-1, 1)
    return torch.from_numpy(np.ascontiguousarray(a.T)).cuda().t()


def run_group(utv, handles, A, B, b, q, seed):
    P = len(handles)
    m, n = A.shape
    Ad = dev(A)
    shards = [utv.colmajor(D.scatter_columns(Ad, b, P, p).clone()) for p in range(P)]
    for p in range(P):
        assert shards[p].shape[1] == utv.dist_local_cols(n, b, P, p)
    Bs = [dev(B) for _ in range(P)]
    Xs = [utv.colmajor_empty(n, Bs[0].shape[1]) for _ in range(P)]
    torch.cuda.synchronize()
    out = [None] * P
    err = [None] * P
    opts = utv.Opts(block=b, power_iters=q, tau=1e-10, seed=seed)

    def work(p):
        try:
            Ap = shards[p] if shards[p].shape[1] > 0 else utv.colmajor_empty(m, 1)
            out[p] = handles[p].lstsq(Ap, Bs[p], Xs[p], opts)
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
    return [X.cpu().numpy() for X in Xs], out


@pytest.mark.parametrize("P,m,n,r,b,q,k", [
    (2, 600, 600, 300, 64, 1, 2),
    (3, 700, 550, 260, 64, 2, 3),     # ragged last block
    (4, 300, 300, 150, 32, 1, 1),
    (5, 130, 100, 40, 32, 1, 1),      # more ranks than blocks: rank 4 holds no column
    (2, 2048, 2048, 1000, 256, 2, 1),
])
def test_local_group_matches_oracle(utv, P, m, n, r, b, q, k):
    M = gen.GpMatrix(m, n, r, seed=m + n + P)
    B, X0 = M.known_rhs(k=k)
    B = B.reshape(m, -1)
    Xo, ro = oracle.lstsq(M.A, B, b=b, q=q, tau=1e-10, seed=11)
    hs = utv.local_group(P)
    try:
        Xs, rs = run_group(utv, hs, M.A, B, b, q, 11)
    finally:
        for h in hs:
            h.close()
    assert all(x == ro == r for x in rs), (rs, ro)
    for X in Xs:
        assert np.array_equal(X, Xs[0])                     # replicated result, bit-identical
    assert np.linalg.norm(Xs[0] - Xo) <= 1e-9 * np.linalg.norm(Xo)
    assert np.linalg.norm(Xs[0] - X0) <= 1e-10 * np.linalg.norm(X0)


def test_local_group_single_rank_equals_in_core(utv):
    """P = 1: the multi-GPU orchestration with no peers == the single-GPU path (rounding only)."""
    m, n, r, b, q = 900, 700, 333, 128, 2
    M = gen.GpMatrix(m, n, r, seed=2)
    B, _ = M.known_rhs(k=2)
    hs = utv.local_group(1)
    try:
        Xs, rs = run_group(utv, hs, M.A, B, b, q, 4)
    finally:
        hs[0].close()
    Xd, rd = utv.lstsq(dev(M.A), dev(B), utv.Opts(block=b, power_iters=q, tau=1e-10, seed=4))
    Xd = Xd.cpu().numpy()
    assert rs[0] == rd == r
    assert np.linalg.norm(Xs[0] - Xd) <= 1e-12 * np.linalg.norm(Xd)


def test_nccl_single_rank(utv):
    """utv_create_dist through NCCL (nranks = 1 on the one GPU available)."""
    uid = utv.get_unique_id()
    assert len(uid) == 128
    h = utv.dist_handle(uid, 1, 0)
    try:
        m, n, r, b = 500, 400, 180, 64
        M = gen.GpMatrix(m, n, r, seed=8)
        B, X0 = M.known_rhs(k=1)
        Xo, ro = oracle.lstsq(M.A, B, b=b, q=1, tau=1e-10, seed=3)
        Xs, rs = run_group(utv, [h], M.A, B.reshape(m, 1), b, 1, 3)
    finally:
        h.close()
    assert rs[0] == ro == r
    assert np.linalg.norm(Xs[0] - Xo) <= 1e-9 * np.linalg.norm(Xo)


def test_dist_handle_rejects_unsupported_flags(utv):
    hs = utv.local_group(1)
    h = hs[0]
    try:
        A = utv.colmajor_empty(64, 64).zero_()
        U = utv.colmajor_empty(64, 64)
        with pytest.raises(utv.UtvError) as e:
            h.factor(A, U=U, opts=utv.Opts(block=16, flags=utv.UTV_WANT_U), n=64)
        assert e.value.status == utv.UTV_ERR_UNSUPPORTED
        B = utv.colmajor_empty(64, 1).zero_()
        X = utv.colmajor_empty(64, 1)
        with pytest.raises(utv.UtvError) as e:
            h.lstsq(A, B, X, utv.Opts(block=16, flags=utv.UTV_NULLIFY_T12))
        assert e.value.status == utv.UTV_ERR_UNSUPPORTED
    finally:
        h.close()


def test_local_group_failing_rank_releases_peers(utv):
    """A rank whose call fails its checks (bad argument) fails the call on EVERY rank: the ranks
    agree on the call (one AllReduce of a flag) before the first collective of the method, so
    the peer gets an error instead of blocking in a collective, and the group stays usable
    (a rank-local failure must not leave the peers hanging)."""
    import oracle
    import utv_inputs as gen
    hs = utv.local_group(2)
    try:
        m, n, b = 256, 256, 64
        M = gen.GpMatrix(m, n, 100, seed=5)
        Bn, _ = M.known_rhs(k=1)
        st = [None, None]

        def run(taus):
            Ad = dev(M.A)
            A = [utv.colmajor(D.scatter_columns(Ad, b, 2, p).clone()) for p in range(2)]
            B = [dev(Bn) for _ in range(2)]
            X = [utv.colmajor_empty(n, 1) for _ in range(2)]
            torch.cuda.synchronize()

            def work(p):
                try:
                    st[p] = hs[p].lstsq(A[p], B[p], X[p], utv.Opts(block=b, power_iters=1, tau=taus[p]))
                except utv.UtvError as e:
                    st[p] = ("err", e.status)

            ts = [threading.Thread(target=work, args=(p,)) for p in range(2)]
            for t in ts:
                t.start()
            for t in ts:
                t.join(timeout=120)
            assert not any(t.is_alive() for t in ts), "a rank hung"
            return X

        run([1e-10, 2.0])                                    # rank 1: tau outside [0, 1) -> UTV_ERR_ARG
        assert st[0] == ("err", utv.UTV_ERR_ARG) and st[1] == ("err", utv.UTV_ERR_ARG), st
        X = run([1e-10, 1e-10])                              # the same group, a valid call
        Xo, ro = oracle.lstsq(M.A, Bn, b=b, q=1, tau=1e-10, seed=1)
        assert st == [ro, ro] == [100, 100]
        for Xp in X:
            assert np.linalg.norm(Xp.cpu().numpy() - Xo) <= 1e-9 * np.linalg.norm(Xo)
    finally:
        for h in hs:
            h.close()


def test_local_group_nan_on_one_rank_fails_all(utv):
    """NaN in one rank's shard: the finiteness flags are AllReduce-d, every rank returns
    UTV_ERR_NUMERICAL (utv.h), none hangs."""
    hs = utv.local_group(2)
    try:
        m, n, b = 200, 192, 64
        rng = np.random.default_rng(3)
        A = [utv.colmajor(dev(rng.standard_normal((m, utv.dist_local_cols(n, b, 2, p))))) for p in range(2)]
        A[1][5, 7] = float("nan")
        B = [dev(np.ones((m, 1))) for _ in range(2)]
        X = [utv.colmajor_empty(n, 1) for _ in range(2)]
        torch.cuda.synchronize()
        st = [None, None]

        def work(p):
            try:
                hs[p].lstsq(A[p], B[p], X[p], utv.Opts(block=b, power_iters=1))
                st[p] = 0
            except utv.UtvError as e:
                st[p] = e.status

        ts = [threading.Thread(target=work, args=(p,)) for p in range(2)]
        for t in ts:
            t.start()
        for t in ts:
            t.join(timeout=120)
        assert not any(t.is_alive() for t in ts), "a rank hung"
        assert st == [utv.UTV_ERR_NUMERICAL, utv.UTV_ERR_NUMERICAL], st
    finally:
        for h in hs:
            h.close()


@pytest.mark.parametrize("P,chunks,lag", [(2, 1, 1), (2, 3, 5), (3, 4, 8), (3, 2, 2), (1, 2, 8)])
def test_local_group_chunks_and_svd_lag(utv, P, chunks, lag):
    """The overlap schedule of the multi-GPU path: the power-iteration and X = A W_V
    products in `chunks` column chunks (each chunk's AllReduce on the communication stream) and
    the SVD of a diagonal block applied `lag` steps after its panel QR.  Against the oracle (x to
    1e-9, r identical).  A later U_s^T / V_s only reorders commuting factors (reading H5), so X
    agrees with lag 1 to rounding."""
    m, n, r, b, q, k = 700, 650, 300, 64, 2, 2
    M = gen.GpMatrix(m, n, r, seed=31 + P)
    B, X0 = M.known_rhs(k=k)
    Xo, ro = oracle.lstsq(M.A, B, b=b, q=q, tau=1e-10, seed=5)
    res = {}
    for lg in sorted({1, lag}):
        hs = utv.local_group(P)
        try:
            with utv.tuned(utv.UTV_TUNE_DIST_CHUNKS, chunks), utv.tuned(utv.UTV_TUNE_SVD_LAG, lg):
                Xs, rs = run_group(utv, hs, M.A, B, b, q, 5)
        finally:
            for h in hs:
                h.close()
        assert all(x == ro == r for x in rs), (rs, ro)
        for X in Xs:
            assert np.array_equal(X, Xs[0])
        assert np.linalg.norm(Xs[0] - Xo) <= 1e-9 * np.linalg.norm(Xo)
        res[lg] = Xs[0]
    assert np.linalg.norm(res[1] - res[lag]) <= 1e-12 * np.linalg.norm(res[1])


@pytest.mark.parametrize("P,m,n,r,b,q,k", [(2, 600, 520, 250, 64, 1, 2), (3, 700, 700, 300, 64, 2, 1),
                                          (1, 500, 400, 180, 64, 1, 1)])
def test_local_group_factor(utv, P, m, n, r, b, q, k):
    """utv_factor on a multi-GPU handle (SURVEY 8(b) distributed mode): every rank's shard of T,
    its contiguous row block of V and the replicated C = U^T B.  Gathered, they satisfy: V orthogonal,
    ||(A V)_j|| = ||T_j|| per column (A V = U T), T zero below the diagonal, and x = V(:, 0:r)
    T11^{-1} C(0:r) equal to the oracle's least-squares solution (1e-9); rank identical."""
    M = gen.GpMatrix(m, n, r, seed=m + n + 7 * P)
    B, _ = M.known_rhs(k=k)
    B = B.reshape(m, -1)
    Xo, ro = oracle.lstsq(M.A, B, b=b, q=q, tau=1e-10, seed=6)
    Ad = dev(M.A)
    hs = utv.local_group(P)
    per = (n + P - 1) // P
    try:
        shards = [utv.colmajor(D.scatter_columns(Ad, b, P, p).clone()) for p in range(P)]
        Bs = [dev(B) for _ in range(P)]
        Vs = [utv.colmajor_empty(max(1, min(n, (p + 1) * per) - min(n, p * per)), n) for p in range(P)]
        torch.cuda.synchronize()
        out, err = [None] * P, [None] * P

        def work(p):
            try:
                Ap = shards[p] if shards[p].shape[1] > 0 else utv.colmajor_empty(m, 1)
                out[p] = hs[p].factor(Ap, V=Vs[p], B=Bs[p], opts=utv.Opts(block=b, power_iters=q, tau=1e-10, seed=6),
                                      n=n)
            except Exception as e:          # noqa: BLE001
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
        T = D.gather_columns(shards, n, b).cpu().numpy()
        V = np.vstack([Vs[p][:min(n, (p + 1) * per) - min(n, p * per)].cpu().numpy() for p in range(P)])
        C = Bs[0].cpu().numpy()
        for Bp in Bs[1:]:
            assert np.array_equal(Bp.cpu().numpy(), C)                  # replicated U^T B
    finally:
        for h in hs:
            h.close()
    assert out == [ro] * P and ro == r, (out, ro)
    assert np.abs(V.T @ V - np.eye(n)).max() <= 1e-13
    assert np.all(np.tril(T, -1) == 0.0)
    AV = M.A @ V
    nrm_av, nrm_t = np.linalg.norm(AV, axis=0), np.linalg.norm(T, axis=0)
    assert np.abs(nrm_av - nrm_t).max() <= 1e-12 * np.linalg.norm(M.A)
    z = np.linalg.solve(T[:r, :r], C[:r])
    X = V[:, :r] @ z
    assert np.linalg.norm(X - Xo) <= 1e-9 * np.linalg.norm(Xo)


def test_local_group_factor_then_solve(utv):
    """utv_factor then utv_solve on a multi-GPU handle: the distributed block back substitution on
    the T shards, X's row blocks from the V row blocks, AllGather -- X replicated, equal on every
    rank and to the oracle's solution."""
    P, m, n, r, b, q = 3, 650, 600, 270, 64, 1
    M = gen.GpMatrix(m, n, r, seed=99)
    B, _ = M.known_rhs(k=2)
    Xo, ro = oracle.lstsq(M.A, B, b=b, q=q, tau=1e-10, seed=2)
    Ad = dev(M.A)
    hs = utv.local_group(P)
    per = (n + P - 1) // P
    try:
        shards = [utv.colmajor(D.scatter_columns(Ad, b, P, p).clone()) for p in range(P)]
        Bs = [dev(B) for _ in range(P)]
        Vs = [utv.colmajor_empty(max(1, min(n, (p + 1) * per) - min(n, p * per)), n) for p in range(P)]
        Xs = [utv.colmajor_empty(n, 2) for _ in range(P)]
        rk = [None] * P
        err = [None] * P

        def work(p):
            try:
                rk[p] = hs[p].factor(shards[p], V=Vs[p], B=Bs[p], opts=utv.Opts(block=b, power_iters=q, tau=1e-10,
                                                                                    seed=2), n=n)
                hs[p].solve(shards[p], Vs[p], Bs[p], rk[p], Xs[p])
            except Exception as e:          # noqa: BLE001
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
        X = [x.cpu().numpy() for x in Xs]
    finally:
        for h in hs:
            h.close()
    assert rk == [ro] * P and ro == r
    for x in X:
        assert np.array_equal(x, X[0])
    assert np.linalg.norm(X[0] - Xo) <= 1e-9 * np.linalg.norm(Xo)


def test_local_group_cholqr_forced(utv):
    """The multi-GPU path (QR(Y) on every rank, the owner's a5 panel) with CholeskyQR2 panels forced
    (R22): X bit-identical on every rank, x to 1e-9 of the oracle, r identical."""
    with utv.tuned(utv.UTV_TUNE_QR_CHOLQR, 2):
        test_local_group_matches_oracle(utv, 3, 700, 550, 260, 64, 2, 3)
