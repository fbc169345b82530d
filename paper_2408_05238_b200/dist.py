"""Multi-GPU randUTV least squares: one process per GPU, block-cyclic columns.

Layout:
* A (m x n) is split into column blocks of width b; block j lives on rank j mod P, and each rank
  stores its blocks packed in order (column-major, ld = m): ``scatter_columns``.
* V (n x n) is split into contiguous row blocks of ceil(n/P) rows: every V update is a right
  multiplication by a replicated factor, so V needs no communication.
* B / C = U^T B (m x k) and the small factors (G, W_V, T_V, W_U, T_U, U_s, V_s) are replicated;
  the Philox sketch is counter-based, so every rank draws the same G without communication.

One step of fig:alg_utv per block column i (owner o = i mod P):
  Z = sum_p A'_p Y_p              AllReduce (m' x b), q times       [a2]
  Y = rows of all ranks           AllGather (n' x b); every rank runs the same QR(Y)  [a3]
  X = sum_p A_p W_V,p             AllReduce (m x b); local right update of A and V     [a4]
  panel QR on o                   Broadcast (W_U, T_U)                                 [a5]
  local left update of A, C                                                            [a6]
  SVD of R on o                   Broadcast (U_s, V_s); local A12 / V1 / C1 updates    [a7]
then Compute_rank on the AllReduce-d diagonal (a8) and the block back substitution with one
AllReduce + Broadcast of b x k per block, X = V z with an AllGather of the row blocks (a9).

The arithmetic of every step runs in the ``steps`` backend: ``CudaSteps`` (the product: the
sm_100a kernels of libutv.so through its step-level C ABI, collectives over NCCL via
torch.distributed).  Orchestration and the collectives are plumbing (index bookkeeping,
memcpy-like gathers).  The CPU tests drive the same orchestration with a CPU backend over gloo.
"""
from __future__ import annotations

import bisect
import math

import torch
import torch.distributed as dist


# ----------------------------------------------------------------------------- layout helpers
def my_blocks(nblocks: int, P: int, p: int):
    return list(range(p, nblocks, P))


def block_width(blk: int, n: int, b: int) -> int:
    return min(b, n - blk * b)


def local_ncols(n: int, b: int, P: int, p: int) -> int:
    return sum(block_width(blk, n, b) for blk in my_blocks(math.ceil(n / b), P, p))


def _colmajor_like(rows, cols, ref: torch.Tensor):
    return torch.empty((cols, rows), dtype=ref.dtype, device=ref.device).t()


def scatter_columns(A: torch.Tensor, b: int, P: int, p: int) -> torch.Tensor:
    """This rank's block-cyclic column shard of A (column-major copy)."""
    m, n = A.shape
    out = _colmajor_like(m, local_ncols(n, b, P, p), A)
    c = 0
    for blk in my_blocks(math.ceil(n / b), P, p):
        w = block_width(blk, n, b)
        out[:, c:c + w].copy_(A[:, blk * b: blk * b + w])
        c += w
    return out


def gather_columns(shards, n: int, b: int) -> torch.Tensor:
    """Inverse of scatter_columns (shards = list indexed by rank)."""
    P = len(shards)
    m = shards[0].shape[0]
    out = _colmajor_like(m, n, shards[0])
    for p in range(P):
        c = 0
        for blk in my_blocks(math.ceil(n / b), P, p):
            w = block_width(blk, n, b)
            out[:, blk * b: blk * b + w].copy_(shards[p][:, c:c + w])
            c += w
    return out


# ----------------------------------------------------------------------------- product backend
class CudaSteps:
    """The sm_100a kernels of libutv.so, step by step (utv_steps.h)."""

    def __init__(self, handle=None):
        import paper_2408_05238_b200 as utv
        self.utv = utv
        self.h = handle or utv.default_handle()
        self.device = torch.device(f"cuda:{self.h.device}")

    def empty(self, rows, cols):
        return torch.empty((cols, rows), dtype=torch.float64, device=self.device).t()

    def zeros(self, rows, cols):
        return torch.zeros((cols, rows), dtype=torch.float64, device=self.device).t()

    def sketch(self, seed, step, row0, mrows, b):
        return self.h.sketch(seed, step, row0, mrows, b)

    def gemm(self, ta, tb, alpha, A, B, beta, Cm):
        self.h.gemm(ta, tb, alpha, A, B, beta, Cm)

    def hqr(self, P):
        """P in place -> R (upper) / zeros; returns (W, T)."""
        _, W, _, T = self.h.hqr(P)
        return W, T

    def svd_block(self, A11):
        Us, _, Vs = self.h.svd_block(A11)
        return Us, Vs

    def trsm_upper(self, T, Z):
        self.h.trsm_upper(T, Z)

    def rank_diag(self, d, tau):
        return self.h.rank_diag(d, tau)

    def finish(self):
        failed, _ = self.h.svd_status()
        if failed:
            raise self.utv.UtvError(self.utv.UTV_ERR_NUMERICAL, "Jacobi SVD did not converge in 30 sweeps")


# ----------------------------------------------------------------------------- collectives
def _allreduce(t, group):
    # column-major tensors are the transpose of a contiguous buffer
    dist.all_reduce(t.t() if not t.is_contiguous() else t, group=group)


def _broadcast(t, src, group):
    dist.broadcast(t.t() if not t.is_contiguous() else t, src=src, group=group)


def _allgather_rows(local, P, group):
    """local: column-major (L x c) padded to the same L on every rank -> list of P (L x c)."""
    L, c = local.shape
    flat = local.t().contiguous().reshape(-1)
    out = torch.empty(P * flat.numel(), dtype=flat.dtype, device=flat.device)
    dist.all_gather_into_tensor(out, flat, group=group)
    return [out[q * flat.numel():(q + 1) * flat.numel()].reshape(c, L).t() for q in range(P)]


# ----------------------------------------------------------------------------- the algorithm
def lstsq_dist(A_loc: torch.Tensor, B: torch.Tensor, n: int, b: int = 256, q: int = 2, tau: float = 1e-10,
               seed: int = 1, steps=None, group=None):
    """x_simple for min ||A x - B|| on P ranks (fast option).

    A_loc: this rank's block-cyclic column shard (scatter_columns), consumed (becomes T's shard).
    B: the full m x k right-hand side (replicated, not modified).  Returns (X (n x k, replicated), r).
    """
    steps = steps or CudaSteps()
    P = dist.get_world_size(group) if dist.is_initialized() else 1
    p = dist.get_rank(group) if dist.is_initialized() else 0
    m = A_loc.shape[0]
    k = B.shape[1] if B.dim() == 2 else 1
    nb = math.ceil(n / b)
    blocks = my_blocks(nb, P, p)
    pos = {blk: t for t, blk in enumerate(blocks)}
    lcol = lambda blk: pos[blk] * b                       # every block but the global last is b wide
    nv = math.ceil(n / P)
    v0 = p * nv
    V = steps.zeros(nv, n)                                  # this rank's rows of V = I
    if v0 < n:
        V[:, v0:min(n, v0 + nv)].diagonal().fill_(1.0)
    Cm = steps.empty(m, k)
    Cm.copy_(B.reshape(m, k))

    for i in range(nb):
        j0 = i * b
        bw = block_width(i, n, b)
        mp, np_ = m - j0, n - j0
        own = i % P
        first = bisect.bisect_left(blocks, i)
        trail = blocks[first:]                             # my blocks >= i
        lt = first * b
        ncl = sum(block_width(blk, n, b) for blk in trail)
        rest = trail[1:] if trail and trail[0] == i else trail   # my blocks > i
        lr = lt + (bw if trail and trail[0] == i else 0)
        nrl = ncl - (bw if trail and trail[0] == i else 0)

        if np_ > b:                                        # R5: no sketch for the last block
            G = steps.sketch(seed, i, j0, mp, b)           # a1 (identical on every rank)
            Yl = steps.zeros(ncl, b)
            if ncl:
                steps.gemm(True, False, 1.0, A_loc[j0:, lt:lt + ncl], G, 0.0, Yl)
            for _ in range(q):                             # a2
                Z = steps.zeros(mp, b)
                if ncl:
                    steps.gemm(False, False, 1.0, A_loc[j0:, lt:lt + ncl], Yl, 0.0, Z)
                if P > 1:
                    _allreduce(Z, group)
                if ncl:
                    steps.gemm(True, False, 1.0, A_loc[j0:, lt:lt + ncl], Z, 0.0, Yl)
            # AllGather the row blocks of Y into global order (padded to the max per rank)
            Lmax = math.ceil((nb - i) / P) * b
            Ypad = steps.zeros(Lmax, b)
            Ypad[:ncl].copy_(Yl)
            parts = _allgather_rows(Ypad, P, group) if P > 1 else [Ypad]
            Y = steps.empty(np_, b)
            cnt = [0] * P
            for blk in range(i, nb):
                o, w = blk % P, block_width(blk, n, b)
                Y[blk * b - j0: blk * b - j0 + w].copy_(parts[o][cnt[o]:cnt[o] + w])
                cnt[o] += w
            Wv, Tv = steps.hqr(Y)                          # a3: identical on every rank
            Wl = steps.empty(ncl, b)                       # rows of W_V for my trailing columns
            c = 0
            for blk in trail:
                w = block_width(blk, n, b)
                Wl[c:c + w].copy_(Wv[blk * b - j0: blk * b - j0 + w])
                c += w
            X = steps.zeros(m, b)                          # a4, R1: all rows
            if ncl:
                steps.gemm(False, False, 1.0, A_loc[:, lt:lt + ncl], Wl, 0.0, X)
            if P > 1:
                _allreduce(X, group)
            X2 = steps.empty(m, b)
            steps.gemm(False, False, 1.0, X, Tv, 0.0, X2)
            if ncl:
                steps.gemm(False, True, -1.0, X2, Wl, 1.0, A_loc[:, lt:lt + ncl])
            Xv = steps.empty(nv, b)                        # V rows (local)
            steps.gemm(False, False, 1.0, V[:, j0:], Wv, 0.0, Xv)
            Xv2 = steps.empty(nv, b)
            steps.gemm(False, False, 1.0, Xv, Tv, 0.0, Xv2)
            steps.gemm(False, True, -1.0, Xv2, Wv, 1.0, V[:, j0:])

        # ---- a5: panel QR on the owner, Broadcast (W_U, T_U)
        Wu = steps.empty(mp, bw)
        Tu = steps.empty(bw, bw)
        if p == own:
            c0 = lcol(i)
            Wq, Tq = steps.hqr(A_loc[j0:, c0:c0 + bw])
            Wu.copy_(Wq)
            Tu.copy_(Tq)
        if P > 1:
            _broadcast(Wu, own, group)
            _broadcast(Tu, own, group)
        # ---- a6: left update of my blocks > i, and of the replicated C
        if nrl:
            Ar = A_loc[j0:, lr:lr + nrl]
            Z1 = steps.empty(bw, nrl)
            steps.gemm(True, False, 1.0, Wu, Ar, 0.0, Z1)
            Z2 = steps.empty(bw, nrl)
            steps.gemm(True, False, 1.0, Tu, Z1, 0.0, Z2)
            steps.gemm(False, False, -1.0, Wu, Z2, 1.0, Ar)
        Z1 = steps.empty(bw, k)
        steps.gemm(True, False, 1.0, Wu, Cm[j0:], 0.0, Z1)
        Z2 = steps.empty(bw, k)
        steps.gemm(True, False, 1.0, Tu, Z1, 0.0, Z2)
        steps.gemm(False, False, -1.0, Wu, Z2, 1.0, Cm[j0:])
        # ---- a7: SVD on the owner, Broadcast (U_s, V_s), local updates
        Us = steps.empty(bw, bw)
        Vs = steps.empty(bw, bw)
        if p == own:
            c0 = lcol(i)
            Uq, Vq = steps.svd_block(A_loc[j0:j0 + bw, c0:c0 + bw])
            Us.copy_(Uq)
            Vs.copy_(Vq)
            if j0 > 0:                                     # A01 := A01 V_s
                tmp = steps.empty(j0, bw)
                steps.gemm(False, False, 1.0, A_loc[:j0, c0:c0 + bw], Vs, 0.0, tmp)
                A_loc[:j0, c0:c0 + bw].copy_(tmp)
        if P > 1:
            _broadcast(Us, own, group)
            _broadcast(Vs, own, group)
        if nrl:                                            # A12 := U_s^T A12
            tmp = steps.empty(bw, nrl)
            steps.gemm(True, False, 1.0, Us, A_loc[j0:j0 + bw, lr:lr + nrl], 0.0, tmp)
            A_loc[j0:j0 + bw, lr:lr + nrl].copy_(tmp)
        tmp = steps.empty(nv, bw)                          # V1 := V1 V_s
        steps.gemm(False, False, 1.0, V[:, j0:j0 + bw], Vs, 0.0, tmp)
        V[:, j0:j0 + bw].copy_(tmp)
        tmp = steps.empty(bw, k)                           # C1 := U_s^T C1
        steps.gemm(True, False, 1.0, Us, Cm[j0:j0 + bw], 0.0, tmp)
        Cm[j0:j0 + bw].copy_(tmp)
    steps.finish()

    # ---- a8: Compute_rank on the diagonal gathered from the column owners
    d = torch.zeros(n, dtype=torch.float64, device=A_loc.device)
    for blk in blocks:
        w = block_width(blk, n, b)
        c0 = lcol(blk)
        d[blk * b: blk * b + w].copy_(torch.diagonal(A_loc[blk * b: blk * b + w, c0:c0 + w]))
    if P > 1:
        dist.all_reduce(d, group=group)
    r = steps.rank_diag(d, tau)

    # ---- a9: z = T11^{-1} C(0:r, :) block by block from the bottom, X = V(:, 0:r) z
    z = steps.zeros(max(r, 1), k)
    S = steps.zeros(max(r, 1), k)                          # this rank's partial sums T[:, blk] z_blk
    if r > 0:
        eye = steps.zeros(b, b)
        eye.diagonal().fill_(1.0)
        for blk in range((r - 1) // b, -1, -1):
            j0, j1 = blk * b, min(r, blk * b + b)
            w = j1 - j0
            o = blk % P
            s = S[j0:j1].clone()
            if P > 1:
                _allreduce(s, group)
            zb = steps.empty(w, k)
            if p == o:
                c0 = lcol(blk)
                zb.copy_(Cm[j0:j1])
                steps.gemm(False, False, -1.0, eye[:w, :w], s, 1.0, zb)      # C_blk - sum_l T_blk,l z_l
                steps.trsm_upper(A_loc[j0:j1, c0:c0 + w], zb)
                if j0 > 0:
                    steps.gemm(False, False, 1.0, A_loc[:j0, c0:c0 + w], zb, 1.0, S[:j0])
            if P > 1:
                _broadcast(zb, o, group)
            z[j0:j1].copy_(zb)
    Xl = steps.zeros(nv, k)
    if r > 0:
        steps.gemm(False, False, 1.0, V[:, :r], z[:r], 0.0, Xl)
    if P > 1:
        parts = _allgather_rows(Xl, P, group)
        X = steps.empty(P * nv, k)
        for q_ in range(P):
            X[q_ * nv:(q_ + 1) * nv].copy_(parts[q_])
        X = X[:n]
    else:
        X = Xl[:n]
    return X, r
