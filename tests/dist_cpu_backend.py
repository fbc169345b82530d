"""CPU step backend for the multi-GPU orchestration tests (TEST INFRASTRUCTURE).

Drives paper_2408_05238_b200.dist.lstsq_dist with the oracle's step functions on CPU tensors,
so the block-cyclic layout and the collective schedule can be checked with gloo, world_size > 1,
on a machine without GPUs.  The product backend is dist.CudaSteps (libutv kernels over NCCL).
"""
import numpy as np
import torch

import oracle


def cm(rows, cols):
    return torch.empty((cols, rows), dtype=torch.float64).t()


class CpuSteps:
    device = torch.device("cpu")

    def empty(self, rows, cols):
        return cm(rows, cols)

    def zeros(self, rows, cols):
        return torch.zeros((cols, rows), dtype=torch.float64).t()

    def sketch(self, seed, step, row0, mrows, b):
        G = cm(mrows, b)
        G.copy_(torch.from_numpy(oracle.gauss(seed, step, row0, mrows, b)))
        return G

    def gemm(self, ta, tb, alpha, A, B, beta, C):
        prod = (A.t() if ta else A) @ (B.t() if tb else B)
        C.copy_(alpha * prod + (beta * C if beta != 0.0 else 0.0))

    def hqr(self, P):
        m, w = P.shape
        packed, tau, T = oracle.hqr(P.numpy())
        R = np.triu(packed)
        P.copy_(torch.from_numpy(np.where(np.arange(m)[:, None] <= np.arange(w)[None, :], R, 0.0)))
        W = np.tril(packed, -1)
        W[np.arange(w), np.arange(w)] = 1.0
        Wt, Tt = cm(m, w), cm(w, w)
        Wt.copy_(torch.from_numpy(W)); Tt.copy_(torch.from_numpy(T))
        return Wt, Tt

    def svd_block(self, A11):
        Us, s, Vs, _ = oracle.svd_small(A11.numpy())
        A11.copy_(torch.from_numpy(np.diag(s)))
        U, V = cm(*Us.shape), cm(*Vs.shape)
        U.copy_(torch.from_numpy(Us)); V.copy_(torch.from_numpy(Vs))
        return U, V

    def trsm_upper(self, T, Z):
        n = Z.shape[0]
        Z.copy_(torch.linalg.solve_triangular(T[:n, :n].contiguous(), Z.contiguous(), upper=True))

    def rank_diag(self, d, tau):
        return oracle.rank(np.diag(d.numpy()), tau)

    def finish(self):
        pass
