"""Replay of one rank's multi-GPU compute schedule on ONE B200 (the scaling model's measured input).

lstsq_dist (csrc/utv_api.cu) runs, on rank p of P, a fixed sequence of kernels whose shapes depend
only on (m, n, b, q, k, P, p): the local sketch / power-iteration products, QR(Y), the X = A W_V
products, the owner's panel QR, the fused two-sided update of the local trailing blocks and the
deferred SVD application.  This tool launches exactly that sequence (utv_gemm / utv_hqr /
utv_sketch through the C ABI, on random data of the right shapes) for every rank p of P, with CUDA
events at the phase boundaries between collectives, and writes the per-step, per-phase device
times as JSON.  tools/scaling_model.py combines them with a collective-cost model into predicted
times at P = 1, 2, 4, 8 (only one GPU exists in this pool, so the collectives cannot be measured).

  python tools/dist_replay.py [--n 50000] [--b 256] [--q 2] [--k 1] [--P 1 2 4 8] [--out f.json]
"""
import argparse
import ctypes as C
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_05238_b200 as utv  # noqa: E402

PHASES = ["pre", "qry", "x", "panel", "update", "apply"]


def local_cols(n, b, P, p):
    return utv.dist_local_cols(n, b, P, p)


def replay_rank(h, ws, src, m, n, b, q, k, P, p, nch):
    """Enqueue rank p's kernel sequence; returns per-step lists of phase events."""
    L = utv.lib()
    st = h.stream
    nb = (n + b - 1) // b
    nloc = local_cols(n, b, P, p)
    base = ws.data_ptr()
    # workspace carve-up (values are random; only shapes and strides matter)
    lda = m
    A = base                                              # m x nloc (ld m)
    off = m * max(nloc, 1)
    def take(cnt):
        nonlocal off
        o = base + 8 * off
        off += (cnt + 31) // 32 * 32
        return o
    G = take(m * b); Z = take(m * b); Yl = take(max(nloc, 1) * b); Y = take(n * b); Xa = take(m * b)
    X2 = take(m * 2 * b); WP = take(max(nloc, 1) * 2 * b); Wv = take(n * b); Tv = take(b * b); tv = take(b)
    Wu = take(m * b); Tu = take(b * b); tu = take(b); S = take(b * b); Z1 = take(b * max(n, k)); Cm = take(m * max(k, 1))
    Us = take(b * b); Tmp = take(max(m, n) * b); Pq = take(max(m, n) * b)
    assert off <= ws.numel(), (off, ws.numel())

    def gemm(ta, tb, M, N, K, Ap, lda_, Bp, ldb_, Cp, ldc, beta=0.0):
        if M <= 0 or N <= 0 or K <= 0:
            return
        st_ = L.utv_gemm(h.h, int(ta), int(tb), M, N, K, C.c_double(1e-3), C.c_void_p(Ap), lda_, C.c_void_p(Bp),
                         ldb_, C.c_double(beta), C.c_void_p(Cp), ldc)
        if st_ != 0:
            raise RuntimeError(f"utv_gemm {ta}{tb} {M}x{N}x{K}: {st_}")

    def refresh(addr, cnt):
        # a dense random panel before every panel QR: the factorization overwrites its input with R
        # (zeros below), and the CholeskyQR2 path declines such panels (tau = 0 columns), so
        # re-factoring the same buffer would time both algorithms (a ~30 us D2D copy at 50000 x 256)
        i0 = (addr - base) // 8
        ws[i0:i0 + cnt].copy_(src[:cnt])

    def hqr(rows, w):
        # the owner's panel QR (m' x bw) on a scratch panel of the same shape
        refresh(Pq, rows * w)
        h.check(L.utv_hqr(h.h, rows, w, C.c_void_p(Pq), rows, C.c_void_p(Wu), rows, C.c_void_p(tu), C.c_void_p(Tu), b))

    steps = []
    for i in range(nb):
        j0 = i * b
        bw, mp, np_ = min(b, n - j0), m - j0, n - j0
        owner = i % P
        own = p == owner
        first = 0 if i <= p else (i - p + P - 1) // P
        lt = first * b
        ncl = nloc - lt
        lr = lt + (bw if own else 0)
        nrl = ncl - (bw if own else 0)
        ldwp = max(ncl, 1)
        right = np_ > b
        ev = {}

        def mark(name):
            e = torch.cuda.Event(enable_timing=True)
            e.record(st)
            ev[name] = e
        mark("start")
        if right:
            h.check(L.utv_sketch(h.h, C.c_uint64(1), i, j0, mp, b, C.c_void_p(G), mp))
            gemm(1, 0, ncl, b, mp, A + 8 * lda * lt, lda, G, mp, Yl, ldwp)
            for _ in range(q):
                for c in range(nch):
                    c0, c1 = b * c // nch, b * (c + 1) // nch
                    gemm(0, 0, mp, c1 - c0, ncl, A + 8 * lda * lt, lda, Yl + 8 * c0 * ldwp, ldwp, Z + 8 * mp * c0, mp)
                for c in range(nch):
                    c0, c1 = b * c // nch, b * (c + 1) // nch
                    gemm(1, 0, ncl, c1 - c0, mp, A + 8 * lda * lt, lda, Z + 8 * mp * c0, mp, Yl + 8 * c0 * ldwp, ldwp)
        mark("pre")
        if right:
            # QR(Y) (n' x b), identical on every rank
            refresh(Y, np_ * b)
            h.check(L.utv_hqr(h.h, np_, b, C.c_void_p(Y), np_, C.c_void_p(Wv), np_, C.c_void_p(tv), C.c_void_p(Tv), b))
        mark("qry")
        if right:
            for c in range(nch):
                c0, c1 = b * c // nch, b * (c + 1) // nch
                gemm(0, 0, m, c1 - c0, ncl, A + 8 * lda * lt, lda, WP + 8 * c0 * ldwp, ldwp, Xa + 8 * m * c0, m)
            gemm(0, 0, m, b, b, Xa, m, Tv, b, X2, m)
            if j0 > 0:
                gemm(0, 1, j0, ncl, b, X2, m, WP, ldwp, A + 8 * lda * lt, lda, 1.0)
            if own:
                gemm(0, 1, mp, bw, b, X2 + 8 * j0, m, WP, ldwp, A + 8 * (lda * lt + j0), lda, 1.0)
        mark("x")
        if own:
            hqr(mp, bw)
        mark("panel")
        if nrl > 0:
            gemm(1, 0, bw, nrl, mp, Wu, mp, A + 8 * (lda * lr + j0), lda, Z1, bw)
            if right:
                gemm(1, 0, bw, b, mp, Wu, mp, X2 + 8 * j0, m, S, bw)
                gemm(0, 1, bw, nrl, b, S, bw, WP, ldwp, Z1, bw, 1.0)
                gemm(1, 0, nrl, bw, bw, Z1, bw, Tu, b, WP + 8 * b * ldwp, ldwp)
                gemm(0, 1, mp, nrl, 2 * b, X2 + 8 * j0, m, WP, ldwp, A + 8 * (lda * lr + j0), lda, 1.0)
            else:
                gemm(1, 0, bw, nrl, bw, Tu, b, Z1, bw, S, bw)
                gemm(0, 0, mp, nrl, bw, Wu, mp, S, bw, A + 8 * (lda * lr + j0), lda, 1.0)
        if k > 0:
            gemm(1, 0, bw, k, mp, Wu, mp, Cm + 8 * j0, m, Z1, bw)
            gemm(1, 0, bw, k, bw, Tu, b, Z1, bw, S, bw)
            gemm(0, 0, mp, k, bw, Wu, mp, S, bw, Cm + 8 * j0, m, 1.0)
        mark("update")
        # deferred SVD application of block i (same shapes whatever the lag)
        if own and j0 > 0:
            gemm(0, 0, j0, bw, bw, A + 8 * lda * lt, lda, Us, b, Tmp, j0)
        if nrl > 0:
            gemm(1, 0, bw, nrl, bw, Us, b, A + 8 * (lda * lr + j0), lda, Tmp, bw)
        if k > 0:
            gemm(1, 0, bw, k, bw, Us, b, Cm + 8 * j0, m, Z1, bw)
        mark("apply")
        steps.append((ev, own, mp, np_))
    return steps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=0)
    ap.add_argument("--n", type=int, default=50000)
    ap.add_argument("--b", type=int, default=256)
    ap.add_argument("--q", type=int, default=2)
    ap.add_argument("--k", type=int, default=1)
    ap.add_argument("--P", type=int, nargs="+", default=[1, 2, 4, 8])
    ap.add_argument("--chunks", type=int, default=2)
    ap.add_argument("--ranks", default="all", help="'all' or a comma list")
    ap.add_argument("--out", default="gpurun_out/dist_replay.json")
    a = ap.parse_args()
    m = a.m or a.n
    n, b, q, k = a.n, a.b, a.q, a.k
    torch.cuda.set_device(0)
    h = utv.Handle(0)
    out = {"m": m, "n": n, "b": b, "q": q, "k": k, "chunks": a.chunks, "phases": PHASES, "runs": []}
    # SVD of one b x b block (side stream work of the owner)
    R = torch.triu(torch.randn(b, b, dtype=torch.float64, device="cuda")).t().contiguous().t()
    h.svd_small(R)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(5):
        e0.record(h.stream)
        h.svd_small(R)
        e1.record(h.stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    out["svd_ms"] = sorted(ts)[len(ts) // 2]
    print("svd_small", out["svd_ms"], "ms", flush=True)
    for P in a.P:
        nloc0 = local_cols(n, b, P, 0)
        need = m * max(nloc0, 1) + 40 * max(m, n) * b + 64 * b * b
        ws = torch.randn(need, dtype=torch.float64, device="cuda") * 1e-3
        src = torch.randn(max(m, n) * b, dtype=torch.float64, device="cuda")
        ranks = range(P) if a.ranks == "all" else [int(x) for x in a.ranks.split(",") if int(x) < P]
        nch = a.chunks if P > 1 else 1
        for p in ranks:
            t0 = time.time()
            steps = replay_rank(h, ws, src, m, n, b, q, k, P, p, nch)
            torch.cuda.synchronize()
            per = []
            for ev, own, mp, np_ in steps:
                names = ["start"] + PHASES
                per.append({"own": own, "mp": mp, "np": np_,
                            **{ph: ev[names[j]].elapsed_time(ev[names[j + 1]]) for j, ph in enumerate(PHASES)}})
            tot = sum(sum(s[ph] for ph in PHASES) for s in per)
            print(f"P={P} p={p}: compute {tot / 1e3:.3f} s (wall {time.time() - t0:.1f} s)", flush=True)
            out["runs"].append({"P": P, "p": p, "chunks": nch, "steps": per, "compute_s": tot / 1e3})
        del ws, src
        torch.cuda.empty_cache()
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    json.dump(out, open(a.out, "w"))
    print("wrote", a.out)


if __name__ == "__main__":
    main()
