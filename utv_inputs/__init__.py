"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NONE of the method's arithmetic (no sketch, no QR of the method,
no SVD, no solve): only the test-matrix and right-hand-side recipes of DESIGN.md
"Input recipe", shaped like the paper's workloads:

* ``gp``  -- the paper's generator: an r x n random block made
  diagonally dominant, replicated with random scale factors to fill m rows.
  Exact rank r, flat spectrum.
* ``gd``  -- decaying spectrum A = Q_L diag(d) Q_R^T, d_i = 10^(-alpha i/(r-1)).
* RHS: known-solution construction b = A x0 + r_perp (min-norm LS solution x0),
  plus the paper's scenario 2 (b = ones) and scenario 4 (10% of the
  entries of b = A x scaled by 0.999).

numpy versions build test inputs on the host; ``gp_torch`` builds the same
recipe on the GPU for the benchmark sizes (different random stream, same law).
"""
from __future__ import annotations

import numpy as np

MATRIX_SEED = 20240809
RHS_SEED = 20240810
SKETCH_SEED = 1


class GpMatrix:
    """A = [c_0 B0; c_1 B0; ...][0:m] with B0 = U[0,1)^{r x n} + n * I_{r,n}, c_0 = 1."""

    def __init__(self, m: int, n: int, r: int, seed: int = MATRIX_SEED):
        assert m >= 1 and n >= 1 and 0 <= r <= min(m, n)
        rng = np.random.default_rng(seed)
        self.m, self.n, self.r = m, n, r
        B0 = rng.random((r, n))
        for i in range(r):
            B0[i, i] += n                     # diagonal dominance
        reps = -(-m // r) if r > 0 else 0
        c = np.concatenate([[1.0], rng.uniform(0.5, 1.5, size=max(reps - 1, 0))]) if r > 0 else np.zeros(0)
        self.B0, self.c = B0, c
        A = np.zeros((m, n), order="F")
        for t in range(reps):
            lo, hi = t * r, min(m, (t + 1) * r)
            A[lo:hi, :] = c[t] * B0[: hi - lo, :]
        self.A = A

    def known_rhs(self, k: int = 1, seed: int = RHS_SEED, consistent: bool = False):
        """b = A x0 + r_perp with x0 = B0^T y in the row space and A^T r_perp = 0.

        r_perp = [c_1 w; -c_0 w; 0 ...] needs two full replicas (m >= 2r).  Returns (B, X0).
        """
        rng = np.random.default_rng(seed)
        m, n, r = self.m, self.n, self.r
        y = rng.standard_normal((r, k))
        X0 = self.B0.T @ y
        B = self.A @ X0
        if not consistent:
            assert m >= 2 * r, "inconsistent known-solution RHS needs two full replicas"
            w = rng.standard_normal((r, k))
            rp = np.zeros((m, k))
            rp[:r] = self.c[1] * w
            rp[r:2 * r] = -self.c[0] * w
            scale = np.linalg.norm(B, axis=0) / np.maximum(np.linalg.norm(rp, axis=0), 1e-300)
            B = B + rp * scale
        return np.asfortranarray(B), X0


def gp(m: int, n: int, r: int, seed: int = MATRIX_SEED) -> np.ndarray:
    return GpMatrix(m, n, r, seed).A


class GdMatrix:
    """A = Q_L diag(d) Q_R^T, Q_L (m x r), Q_R (n x r) orthonormalised Gaussians."""

    def __init__(self, m: int, n: int, r: int, alpha: float = 3.0, seed: int = MATRIX_SEED):
        rng = np.random.default_rng(seed)
        self.m, self.n, self.r = m, n, r
        QL, _ = np.linalg.qr(rng.standard_normal((m, r)))
        QR, _ = np.linalg.qr(rng.standard_normal((n, r)))
        d = 10.0 ** (-alpha * np.arange(r) / max(r - 1, 1)) if r > 0 else np.zeros(0)
        self.QL, self.QR, self.d = QL, QR, d
        self.A = np.asfortranarray((QL * d) @ QR.T)

    def known_rhs(self, k: int = 1, seed: int = RHS_SEED, consistent: bool = False):
        rng = np.random.default_rng(seed)
        y = rng.standard_normal((self.r, k))
        X0 = self.QR @ y
        B = self.A @ X0
        if not consistent:
            w = rng.standard_normal((self.m, k))
            rp = w - self.QL @ (self.QL.T @ w)
            scale = np.linalg.norm(B, axis=0) / np.maximum(np.linalg.norm(rp, axis=0), 1e-300)
            B = B + rp * scale
        return np.asfortranarray(B), X0


def gd(m: int, n: int, r: int, alpha: float = 3.0, seed: int = MATRIX_SEED) -> np.ndarray:
    return GdMatrix(m, n, r, alpha, seed).A


def rhs_ones(m: int, k: int = 1) -> np.ndarray:
    """Scenario 2: b set to ones."""
    return np.ones((m, k), order="F")


def rhs_perturbed(A: np.ndarray, k: int = 1, seed: int = RHS_SEED) -> np.ndarray:
    """Scenario 4: b = A x, x ~ U(0,1), then 10% of b's entries set to 99.9%."""
    rng = np.random.default_rng(seed)
    x = rng.random((A.shape[1], k))
    B = A @ x
    idx = rng.choice(A.shape[0], size=max(1, A.shape[0] // 10), replace=False)
    B[idx] *= 0.999
    return np.asfortranarray(B)


def gp_torch(m: int, n: int, r: int, seed: int = MATRIX_SEED, device="cuda", k: int = 1, out=None):
    """The Gp recipe generated on the device (bench sizes).  Column-major storage:
    returns a tensor `At` of shape (n, m) (row-major n x m == column-major m x n),
    plus (B, X0) with a known min-norm solution X0 (consistent part + r_perp).
    """
    import torch

    g = torch.Generator(device=device)
    g.manual_seed(seed)
    B0 = torch.rand((r, n), generator=g, dtype=torch.float64, device=device)
    B0.diagonal().add_(float(n))
    reps = -(-m // r)
    c = torch.cat([torch.ones(1, dtype=torch.float64, device=device),
                   0.5 + torch.rand(reps - 1, generator=g, dtype=torch.float64, device=device)])
    At = out if out is not None else torch.empty((n, m), dtype=torch.float64, device=device)
    for t in range(reps):
        lo, hi = t * r, min(m, (t + 1) * r)
        At[:, lo:hi].copy_((B0[: hi - lo, :] * c[t]).t())
    y = torch.randn((r, k), generator=g, dtype=torch.float64, device=device)
    X0 = B0.t() @ y                                  # n x k, in the row space
    Bm = torch.empty((m, k), dtype=torch.float64, device=device)
    Ax0 = B0 @ X0                                    # r x k
    for t in range(reps):
        lo, hi = t * r, min(m, (t + 1) * r)
        Bm[lo:hi] = c[t] * Ax0[: hi - lo]
    if m >= 2 * r:
        w = torch.randn((r, k), generator=g, dtype=torch.float64, device=device)
        rp = torch.zeros((m, k), dtype=torch.float64, device=device)
        rp[:r] = c[1] * w
        rp[r:2 * r] = -c[0] * w
        scale = Bm.norm(dim=0) / rp.norm(dim=0)
        Bm = Bm + rp * scale
    return At, Bm, X0
