"""CPU oracle for randUTV + least squares (arXiv 2408.05238) -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_2408_05238_b200``) never imports it and shares no code with it.

The arithmetic lives in plain C (``utv_oracle.c``); this module only marshals
numpy arrays (Fortran order, float64) through ctypes.  See the C file header for
citations and for the pin status of each function.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "utv_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

OK, ERR_ARG, ERR_SHAPE, ERR_ALLOC, ERR_NUMERICAL = 0, -1, -2, -3, -6


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (-O2, no fast-math, OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fno-fast-math", "-fopenmp", "-fPIC", "-shared",
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        d, i64, i32, u64 = C.c_void_p, C.c_int64, C.c_int32, C.c_uint64
        _lib.oracle_philox4x32_10.argtypes = [d, d, d]
        _lib.oracle_gauss.argtypes = [u64, i64, i64, i64, i64, d, i64]
        _lib.oracle_hqr.argtypes = [i64, i64, d, i64, d, d, i64]
        _lib.oracle_svd_small.argtypes = [i64, d, i64, d, i64, d, d, i64, d]
        _lib.oracle_svd_small.restype = C.c_int
        _lib.oracle_randutv.argtypes = [i64, i64, i64, d, i64, d, i64, d, i64, d, i64, i64, i32, u64, d]
        _lib.oracle_randutv.restype = C.c_int
        _lib.oracle_rank.argtypes = [i64, d, i64, C.c_double]
        _lib.oracle_rank.restype = i64
        _lib.oracle_solve.argtypes = [i64, i64, d, i64, d, i64, d, i64, i64, d, i64]
        _lib.oracle_lstsq.argtypes = [i64, i64, i64, d, i64, d, i64, d, i64, i64, i32, C.c_double, u64, d]
        _lib.oracle_lstsq.restype = C.c_int
        _lib.oracle_nullify.argtypes = [i64, i64, d, i64, d, i64]
        _lib.oracle_lstsq_ex.argtypes = [i64, i64, i64, d, i64, d, i64, d, i64, i64, i32, C.c_double, u64, C.c_int, d]
        _lib.oracle_lstsq_ex.restype = C.c_int
        _lib.oracle_set_threads.argtypes = [C.c_int]
        _lib.oracle_get_threads.restype = C.c_int
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _f64(a):
    return np.asfortranarray(np.array(a, dtype=np.float64, copy=True))


def set_threads(n: int) -> None:
    lib().oracle_set_threads(int(n))


def get_threads() -> int:
    return lib().oracle_get_threads()


class OracleError(RuntimeError):
    def __init__(self, status):
        super().__init__(f"oracle status {status}")
        self.status = status


def philox4x32_10(ctr, key):
    c = np.array(ctr, dtype=np.uint32); k = np.array(key, dtype=np.uint32)
    out = np.zeros(4, dtype=np.uint32)
    lib().oracle_philox4x32_10(_p(c), _p(k), _p(out))
    return out


def gauss(seed: int, step: int, row0: int, mrows: int, b: int) -> np.ndarray:
    G = np.zeros((mrows, b), dtype=np.float64, order="F")
    lib().oracle_gauss(seed, step, row0, mrows, b, _p(G), max(mrows, 1))
    return G


def hqr(P):
    """Householder QR in place (dlarfg/dlarft). Returns (packed, tau, T)."""
    P = _f64(P); m, n = P.shape
    tau = np.zeros(n); T = np.zeros((n, n), order="F")
    lib().oracle_hqr(m, n, _p(P), max(m, 1), _p(tau), _p(T), max(n, 1))
    return P, tau, T


def svd_small(R):
    """One-sided Jacobi on R^T (reading R9). Returns (Us, sigma, Vs, sweeps)."""
    R = _f64(R); b = R.shape[0]
    Us = np.zeros((b, b), order="F"); Vs = np.zeros((b, b), order="F"); s = np.zeros(b)
    sw = C.c_int(0)
    st = lib().oracle_svd_small(b, _p(R), max(b, 1), _p(Us), max(b, 1), _p(s), _p(Vs), max(b, 1), C.byref(sw))
    if st != OK:
        raise OracleError(st)
    return Us, s, Vs, sw.value


def randutv(A, b: int, q: int, seed: int, B=None, want_u: bool = False):
    """randUTV (fig:alg_utv). Returns dict(T, V, U?, C?, max_sweeps)."""
    A = _f64(A); m, n = A.shape
    V = np.zeros((n, n), order="F")
    U = np.zeros((m, m), order="F") if want_u else None
    Bc = None if B is None else _f64(np.asarray(B).reshape(m, -1))
    k = 0 if Bc is None else Bc.shape[1]
    sw = C.c_int(0)
    st = lib().oracle_randutv(m, n, k, _p(A), max(m, 1), _p(V), max(n, 1), _p(U), max(m, 1),
                              _p(Bc), max(m, 1), b, q, seed, C.byref(sw))
    if st != OK:
        raise OracleError(st)
    out = {"T": A, "V": V, "max_sweeps": sw.value}
    if want_u:
        out["U"] = U
    if Bc is not None:
        out["C"] = Bc
    return out


def rank(T, tau: float) -> int:
    T = _f64(T)
    return int(lib().oracle_rank(T.shape[1], _p(T), max(T.shape[0], 1), float(tau)))


def solve(T, V, Cm, r: int):
    T = _f64(T); V = _f64(V); Cm = _f64(np.asarray(Cm).reshape(T.shape[0], -1))
    n = V.shape[0]; k = Cm.shape[1]
    X = np.zeros((n, k), order="F")
    lib().oracle_solve(n, r, _p(T), max(T.shape[0], 1), _p(V), max(n, 1), _p(Cm), max(Cm.shape[0], 1), k,
                       _p(X), max(n, 1))
    return X


def nullify(T, V, r: int):
    """Nullify_top_right_part_of_T (fig:alg_nullify_t12): returns (T', V') with T'(0:r, r:n) = 0."""
    T = _f64(T); V = _f64(V); n = V.shape[0]
    lib().oracle_nullify(n, int(r), _p(T), max(T.shape[0], 1), _p(V), max(n, 1))
    return T, V


def lstsq(A, B, b: int, q: int, tau: float = 1e-10, seed: int = 1, nullify: bool = False):
    """randUTV least squares (fig:alg_axb; fast option without Nullify unless nullify=True). Returns (X, r).

    m < n goes through lstsq_wide (reading R21)."""
    A = _f64(A); m, n = A.shape
    if m < n:
        if nullify:
            raise OracleError(ERR_ARG)
        return lstsq_wide(A, B, b, q, tau, seed)
    B2 = _f64(np.asarray(B).reshape(m, -1)); k = B2.shape[1]
    X = np.zeros((n, k), order="F")
    r = C.c_int64(0)
    st = lib().oracle_lstsq_ex(m, n, k, _p(A), max(m, 1), _p(B2), max(m, 1), _p(X), max(n, 1), b, q, float(tau),
                               seed, int(bool(nullify)), C.byref(r))
    if st != OK:
        raise OracleError(st)
    return X, int(r.value)


def lstsq_wide(A, B, b: int, q: int, tau: float = 1e-10, seed: int = 1):
    """Wide least squares, m < n (reading R21 in DESIGN.md).

    The paper defines randUTV for m >= n only (its loop guard is garbled, R4).  For m < n the
    oracle runs randUTV on the tall A^T (n x m): A^T V' = U' T' (eq:UTVdef P:467-473), so
    A = V' T'^T U'^T, and with r from Compute_rank on T' (R10) the solution of
    eq:simplesoln transposes to
        X = U'(:, 0:r) T'(0:r, 0:r)^{-T} V'(:, 0:r)^T B.
    Steps: the C randUTV (explicit U' and V'), then numpy / scipy library primitives.
    """
    from scipy.linalg import solve_triangular
    A = _f64(A); m, n = A.shape
    assert m < n
    B2 = _f64(np.asarray(B).reshape(m, -1)); k = B2.shape[1]
    f = randutv(np.asfortranarray(A.T), b, q, seed, want_u=True)
    T, V, U = f["T"], f["V"], f["U"]
    r = rank(T, tau)
    if r == 0:
        return np.zeros((n, k), order="F"), 0
    c = V[:, :r].T @ B2                                       # V'(:, 0:r)^T B
    z = solve_triangular(T[:r, :r], c, trans="T", lower=False)  # T11^{-T} c
    return np.asfortranarray(U[:, :r] @ z), r
