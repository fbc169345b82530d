"""Multi-GPU x out-of-core (UTV_HOST_STREAMED on a multi-GPU handle; SURVEY 8(e) with 8(f) #1, the
north star's cfg5 regime) against the CPU oracle.

Each rank's block-cyclic shard stays in its pinned host memory and is streamed through the rank's
device (the resident part capped with UTV_OOC_MAX_RESIDENT_COLS); the ranks run as an in-process
group on the one GPU of this pool.  Gates: r identical on every rank and
equal to the oracle's, X bit-identical on every rank and within 1e-9 of the oracle, the T left in
host memory with the oracle's diagonal (R20: singular values, sign-free) and an exactly zero
strictly-lower part (R13), and the same x as the in-core multi-GPU path.
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


def run_group(utv, P, A, B, b, q, seed, streamed, flags=0):
    m, n = A.shape
    Ad = dev(A)
    hs = utv.local_group(P)
    try:
        if streamed:
            shards = []
            for p in range(P):
                sh = D.scatter_columns(Ad, b, P, p)
                t = utv.colmajor_empty(m, sh.shape[1], device="cpu", pin_memory=True)
                t.copy_(sh)
                shards.append(t)
        else:
            shards = [utv.colmajor(D.scatter_columns(Ad, b, P, p).clone()) for p in range(P)]
        Bs = [dev(B) for _ in range(P)]
        Xs = [utv.colmajor_empty(n, Bs[0].shape[1]) for _ in range(P)]
        torch.cuda.synchronize()
        out, err = [None] * P, [None] * P
        opts = utv.Opts(block=b, power_iters=q, tau=1e-10, seed=seed,
                        flags=flags | (utv.UTV_HOST_STREAMED if streamed else 0))

        def work(p):
            try:
                Ap = shards[p]
                if Ap.shape[1] == 0:
                    Ap = utv.colmajor_empty(m, 1, device="cpu" if streamed else "cuda")
                out[p] = hs[p].lstsq(Ap, Bs[p], Xs[p], opts)
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
        stats = [hs[p].stream_stats() for p in range(P)] if streamed else None
        T = D.gather_columns([s.cuda() if streamed else s for s in shards], n, b).cpu().numpy()
        return [X.cpu().numpy() for X in Xs], out, T, stats
    finally:
        for h in hs:
            h.close()


@pytest.mark.parametrize("P,m,n,r,b,q,k,cap", [
    (2, 600, 600, 300, 64, 1, 2, 0),          # every block of every shard streamed
    (3, 700, 550, 260, 64, 2, 3, 64),         # ragged last block, one block resident per rank
    (2, 900, 640, 333, 128, 2, 2, 128),       # b = 128, r inside a block
    (1, 640, 512, 200, 64, 1, 1, 0),          # P = 1: the single-rank group, streamed
    (5, 300, 260, 100, 64, 1, 1, 0),          # more ranks than blocks: rank 4 holds no column
])
def test_dist_streamed_matches_oracle(utv, monkeypatch, P, m, n, r, b, q, k, cap):
    monkeypatch.setenv("UTV_OOC_MAX_RESIDENT_COLS", str(cap))
    M = gen.GpMatrix(m, n, r, seed=m + n + P)
    B, X0 = M.known_rhs(k=k)
    B = B.reshape(m, -1)
    Xo, ro = oracle.lstsq(M.A, B, b=b, q=q, tau=1e-10, seed=9)
    Xs, rs, T, stats = run_group(utv, P, M.A, B, b, q, 9, streamed=True)
    assert all(x == ro == r for x in rs), (rs, ro)
    for X in Xs:
        assert np.array_equal(X, Xs[0])
    assert np.linalg.norm(Xs[0] - Xo) <= 1e-9 * np.linalg.norm(Xo)
    assert np.linalg.norm(Xs[0] - X0.reshape(Xs[0].shape)) <= 1e-10 * np.linalg.norm(X0)
    # T in host memory: exactly zero below the diagonal, the oracle's diagonal (non-negative)
    assert np.all(np.tril(T, -1) == 0.0)
    To = oracle.randutv(M.A, b, q, 9)["T"]
    d, do = np.diag(T), np.diag(To)
    assert np.all(d >= 0.0)
    assert np.abs(d - do).max() <= 1e-12 * do.max()
    # something was actually streamed (every rank with columns moved its shard over the link)
    for p, s in enumerate(stats):
        if D.local_ncols(n, b, P, p) > cap:
            assert s["h2d_bytes"] > 0 and s["d2h_bytes"] > 0


def test_dist_streamed_equals_in_core(utv, monkeypatch):
    """The streamed multi-GPU path == the in-core multi-GPU path (same collectives, different
    update grouping: rounding only)."""
    monkeypatch.setenv("UTV_OOC_MAX_RESIDENT_COLS", "64")
    m, n, r, b, q = 800, 700, 350, 64, 2
    M = gen.GpMatrix(m, n, r, seed=77)
    B, _ = M.known_rhs(k=2)
    Xs, rs, Ts, _ = run_group(utv, 2, M.A, B, b, q, 4, streamed=True)
    Xi, ri, Ti, _ = run_group(utv, 2, M.A, B, b, q, 4, streamed=False)
    assert rs == ri == [r, r]
    assert np.linalg.norm(Xs[0] - Xi[0]) <= 1e-12 * np.linalg.norm(Xi[0])
    assert np.abs(np.abs(np.diag(Ts)) - np.abs(np.diag(Ti))).max() <= 1e-12 * np.abs(np.diag(Ti)).max()


def test_dist_streamed_rejects_device_shard(utv):
    """UTV_HOST_STREAMED on a multi-GPU handle needs the shard in host memory: every rank fails
    with UTV_ERR_ARG (agreed before the first collective), none hangs."""
    hs = utv.local_group(2)
    try:
        st = [None, None]
        A = [utv.colmajor_empty(128, 64).zero_() for _ in range(2)]       # m = 128, n = 128: 64 cols each
        Bs = [utv.colmajor_empty(128, 1).zero_() for _ in range(2)]
        Xs = [utv.colmajor_empty(128, 1) for _ in range(2)]

        def work(p):
            try:
                st[p] = hs[p].lstsq(A[p], Bs[p], Xs[p], utv.Opts(block=64, flags=utv.UTV_HOST_STREAMED))
            except utv.UtvError as e:
                st[p] = e.status

        ts = [threading.Thread(target=work, args=(p,)) for p in range(2)]
        for t in ts:
            t.start()
        for t in ts:
            t.join(timeout=120)
        assert not any(t.is_alive() for t in ts)
        assert st == [utv.UTV_ERR_ARG, utv.UTV_ERR_ARG]
    finally:
        for h in hs:
            h.close()


def test_dist_streamed_cholqr_forced(utv, monkeypatch):
    """Multi-GPU x out-of-core with CholeskyQR2 panels forced (R22): the same parity bar."""
    with utv.tuned(utv.UTV_TUNE_QR_CHOLQR, 2):
        test_dist_streamed_matches_oracle(utv, monkeypatch, 2, 900, 640, 333, 128, 2, 2, 128)
