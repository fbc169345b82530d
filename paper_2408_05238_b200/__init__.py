"""paper_2408_05238_b200 -- B200-native randUTV + least squares (arXiv 2408.05238).

Thin Python binding over the C ABI of ``libutv.so`` (``include/utv.h``, ``include/utv_steps.h``):
argument marshalling only -- every step of the method runs in the sm_100a kernels of
``csrc/``.  There is no CPU fallback: if ``libutv.so`` is missing or the device is not a
CUDA GPU the calls raise.

Matrices are column-major (LAPACK layout), passed as torch tensors of shape (rows, cols)
with ``stride(0) == 1`` (e.g. ``colmajor(torch.empty(...))`` or ``t.t().contiguous().t()``).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libutv.so")

UTV_OK, UTV_ERR_ARG, UTV_ERR_SHAPE, UTV_ERR_ALLOC, UTV_ERR_CUDA = 0, -1, -2, -3, -4
UTV_ERR_NCCL, UTV_ERR_NUMERICAL, UTV_ERR_UNSUPPORTED = -5, -6, -7
UTV_WANT_V, UTV_WANT_U, UTV_NULLIFY_T12, UTV_HOST_STREAMED, UTV_EXPLICIT_V, UTV_KEEP_FACTORS = 1, 2, 4, 8, 16, 32

EXPORTED = ["utv_create", "utv_create_dist", "utv_destroy", "utv_last_error", "utv_set_stream", "utv_synchronize",
            "utv_factor", "utv_solve", "utv_lstsq", "utv_version", "utv_sketch", "utv_philox", "utv_hqr",
            "utv_svd_small", "utv_gemm", "utv_rank", "utv_profile", "utv_profile_read",
            "utv_profile_dump", "utv_svd_block", "utv_svd_status", "utv_trsm_upper",
            "utv_rank_diag", "utv_set_device_budget", "utv_stream_stats", "utv_get_unique_id",
            "utv_create_local_group", "utv_dist_local_cols", "utv_tune", "utv_solve_rhs",
            "utv_create_with_comm"]
PROF_FAMILIES = ["gemm", "panel", "svd", "sketch", "solve", "misc"]


class _ProfEntry(C.Structure):
    _fields_ = [("launches", C.c_int64), ("calls", C.c_int64), ("ms", C.c_double), ("flops", C.c_double),
                ("bytes", C.c_double)]


_AR_CB = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p)
_BC_CB = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_int, C.c_void_p)
_AG_CB = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p)
_AB_CB = C.CFUNCTYPE(None, C.c_void_p)


class _CommOps(C.Structure):
    _fields_ = [("allreduce_sum", _AR_CB), ("broadcast", _BC_CB), ("allgather", _AG_CB), ("abort", _AB_CB),
                ("ctx", C.c_void_p)]


class UtvError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"libutv status {status}: {msg}")
        self.status = status


class _Opts(C.Structure):
    _fields_ = [("block", C.c_int64), ("power_iters", C.c_int32), ("tau", C.c_double), ("seed", C.c_uint64),
                ("flags", C.c_uint32)]


@dataclass
class Opts:
    block: int = 256
    power_iters: int = 2
    tau: float = 1e-10
    seed: int = 1
    flags: int = 0

    def c(self) -> _Opts:
        return _Opts(int(self.block), int(self.power_iters), float(self.tau), int(self.seed), int(self.flags))


_lib = None


def lib() -> C.CDLL:
    """Load libutv.so (raises if it has not been built: no fallback path exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: build it with `python -m paper_2408_05238_b200.build` "
                               "(or __graft_entry__.build()); there is no CPU fallback")
        L = C.CDLL(LIB_PATH)
        p, i64, i32, u64, d = C.c_void_p, C.c_int64, C.c_int32, C.c_uint64, C.c_double
        st = C.c_int
        sig = {
            "utv_create": ([C.POINTER(p), C.c_int, p], st),
            "utv_create_dist": ([C.POINTER(p), C.c_int, p, p, C.c_int, C.c_int], st),
            "utv_destroy": ([p], st),
            "utv_last_error": ([p], C.c_char_p),
            "utv_set_stream": ([p, p], st),
            "utv_synchronize": ([p], st),
            "utv_factor": ([p, i64, i64, p, i64, p, i64, p, i64, p, i64, i64, C.POINTER(_Opts), C.POINTER(i64)], st),
            "utv_solve": ([p, i64, i64, i64, p, i64, p, i64, p, i64, i64, p, i64], st),
            "utv_lstsq": ([p, i64, i64, i64, p, i64, p, i64, p, i64, C.POINTER(_Opts), C.POINTER(i64)], st),
            "utv_version": ([], C.c_char_p),
            "utv_sketch": ([p, u64, i64, i64, i64, i64, p, i64], st),
            "utv_philox": ([p, i64, p, p, p], st),
            "utv_hqr": ([p, i64, i64, p, i64, p, i64, p, p, i64], st),
            "utv_svd_small": ([p, i64, p, i64, p, i64, p, p, i64, C.POINTER(i32)], st),
            "utv_gemm": ([p, C.c_int, C.c_int, i64, i64, i64, d, p, i64, p, i64, d, p, i64], st),
            "utv_rank": ([p, i64, p, i64, d, C.POINTER(i64)], st),
            "utv_profile": ([p, C.c_int], st),
            "utv_profile_read": ([p, p], st),
            "utv_profile_dump": ([p, C.c_char_p], st),
            "utv_svd_block": ([p, i64, p, i64, p, i64, p, p, i64], st),
            "utv_svd_status": ([p, C.POINTER(i32), C.POINTER(i32)], st),
            "utv_trsm_upper": ([p, i64, p, i64, p, i64, i64], st),
            "utv_rank_diag": ([p, i64, p, d, C.POINTER(i64)], st),
            "utv_set_device_budget": ([p, i64], st),
            "utv_get_unique_id": ([p], st),
            "utv_create_local_group": ([p, C.c_int, p, p], st),
            "utv_dist_local_cols": ([i64, i64, C.c_int, C.c_int], i64),
            "utv_stream_stats": ([p, C.POINTER(i64), C.POINTER(i64), C.POINTER(i64)], st),
            "utv_tune": ([C.c_int, i64, C.POINTER(i64)], st),
            "utv_solve_rhs": ([p, i64, i64, i64, p, i64, p, i64, p, i64, C.POINTER(i64)], st),
            "utv_create_with_comm": ([C.POINTER(p), C.c_int, p, C.c_int, C.c_int, C.POINTER(_CommOps)], st),
        }
        for name, (args, res) in sig.items():
            f = getattr(L, name)
            f.argtypes, f.restype = args, res
        _lib = L
    return _lib


def version() -> str:
    return lib().utv_version().decode()


# ----------------------------------------------------------------------------- layout helpers
def colmajor_empty(rows: int, cols: int, device="cuda", dtype=torch.float64, pin_memory=False) -> torch.Tensor:
    """An uninitialised column-major (rows x cols) tensor (storage = cols x rows row-major)."""
    if str(device) == "cpu":
        return torch.empty((cols, rows), dtype=dtype, pin_memory=pin_memory).t()
    return torch.empty((cols, rows), dtype=dtype, device=device).t()


def colmajor(t: torch.Tensor) -> torch.Tensor:
    """Column-major copy (or the tensor itself if already column-major)."""
    if t.dim() == 1:
        t = t.reshape(-1, 1)
    if t.stride(0) == 1 and (t.shape[1] <= 1 or t.stride(1) >= max(1, t.shape[0])):
        return t
    return t.t().contiguous().t()


def _ld(t: torch.Tensor) -> int:
    if t.dim() == 1:
        return max(1, t.shape[0])
    if t.stride(0) != 1 and t.shape[0] > 1:
        raise ValueError("matrix must be column-major (stride(0) == 1); use colmajor()")
    return max(1, t.shape[0], t.stride(1) if t.shape[1] > 1 else 0)


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _check_f64(*ts):
    for t in ts:
        if t is not None and t.dtype != torch.float64:
            raise TypeError("libutv computes in FP64: tensors must be torch.float64")


class Handle:
    """A libutv handle bound to one device and stream (default: torch's current stream)."""

    def __init__(self, device: int | None = None, stream: torch.cuda.Stream | None = None):
        if not torch.cuda.is_available():
            raise RuntimeError("libutv needs a CUDA device (no CPU fallback)")
        self.device = torch.cuda.current_device() if device is None else int(device)
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        h = C.c_void_p()
        self._check(lib().utv_create(C.byref(h), self.device, C.c_void_p(self.stream.cuda_stream)), None)
        self.h = h

    @classmethod
    def _wrap(cls, h: C.c_void_p, device: int, stream) -> "Handle":
        obj = cls.__new__(cls)
        obj.device, obj.stream, obj.h = device, stream, h
        obj.multi = True
        return obj

    def _check(self, status: int, h):
        if status != UTV_OK:
            msg = lib().utv_last_error(h).decode() if h is not None else "utv_create failed"
            raise UtvError(status, msg)

    def check(self, status: int):
        self._check(status, self.h)

    def close(self):
        if getattr(self, "h", None):
            lib().utv_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def synchronize(self):
        self.check(lib().utv_synchronize(self.h))

    # ------------------------------------------------------------------ the boundary calls
    def factor(self, A, V=None, U=None, B=None, opts: Opts | None = None, want_rank: bool = True,
               n: int | None = None):
        """randUTV in place: A -> T; V, U (if given; U needs opts.flags & UTV_WANT_U), B -> U^T B.
        On a multi-GPU handle A is this rank's block-cyclic shard, V (optional) this rank's row block
        of V (ceil(n/P) x n) and n the GLOBAL column count (default V.shape[1])."""
        opts = opts or Opts()
        _check_f64(A, V, U, B)
        m, n_a = A.shape
        if getattr(self, "multi", False):
            n = n if n is not None else (V.shape[1] if V is not None else None)
            if n is None:
                raise ValueError("multi-GPU factor: pass the global n (or V)")
        else:
            n = n_a
        k = 0 if B is None else (B.shape[1] if B.dim() == 2 else 1)
        r = C.c_int64(-1)
        o = opts.c()
        self.check(lib().utv_factor(self.h, m, n, _ptr(A), _ld(A), _ptr(V), _ld(V) if V is not None else 1,
                                    _ptr(U), _ld(U) if U is not None else 1, _ptr(B), _ld(B) if B is not None else 1,
                                    k, C.byref(o), C.byref(r) if want_rank else None))
        return int(r.value) if want_rank else None

    def solve(self, T, V, Cm, r: int, X):
        """X = V(:, 0:r) T11^{-1} C(0:r).  On a multi-GPU handle T is this rank's shard, V its row
        block and the global n is X.shape[0]."""
        _check_f64(T, V, Cm, X)
        m, n = T.shape
        if getattr(self, "multi", False):
            n = X.shape[0]
        k = Cm.shape[1] if Cm.dim() == 2 else 1
        self.check(lib().utv_solve(self.h, m, n, int(r), _ptr(T), _ld(T), _ptr(V), _ld(V), _ptr(Cm), _ld(Cm), k,
                                   _ptr(X), _ld(X)))
        return X

    def lstsq(self, A, B, X, opts: Opts | None = None) -> int:
        """Fast-option LS (A, B consumed).  A, B, X may be device or host tensors.  On a multi-GPU
        handle A is this rank's block-cyclic shard and the global n is X.shape[0]."""
        opts = opts or Opts()
        _check_f64(A, B, X)
        m, n = A.shape
        if getattr(self, "multi", False):
            n = X.shape[0]
        k = B.shape[1] if B.dim() == 2 else 1
        r = C.c_int64(-1)
        o = opts.c()
        self.check(lib().utv_lstsq(self.h, m, n, k, _ptr(A), _ld(A), _ptr(B), _ld(B), _ptr(X), _ld(X), C.byref(o),
                                   C.byref(r)))
        return int(r.value)

    def solve_rhs(self, T, B, X, m: int | None = None) -> int:
        """X = V(:,0:r) T11^{-1} (U^T B)(0:r) for a NEW B with the factors kept by the last call with
        UTV_KEEP_FACTORS (utv_solve_rhs); B is overwritten by U^T B.  T is the T that call left in A
        (on a multi-GPU handle: this rank's shard).  Returns r."""
        _check_f64(T, B, X)
        k = B.shape[1] if B.dim() == 2 else 1
        m = B.shape[0] if m is None else m
        n = X.shape[0]
        r = C.c_int64(-1)
        self.check(lib().utv_solve_rhs(self.h, m, n, k, _ptr(T), _ld(T), _ptr(B), _ld(B), _ptr(X), _ld(X),
                                       C.byref(r)))
        return int(r.value)

    def set_device_budget(self, nbytes: int):
        """HBM budget (bytes) of UTV_HOST_STREAMED calls; 0 = free HBM minus 1 GiB."""
        self.check(lib().utv_set_device_budget(self.h, int(nbytes)))

    def stream_stats(self) -> dict:
        """Host-link traffic of the last UTV_HOST_STREAMED call."""
        a, b, c = C.c_int64(0), C.c_int64(0), C.c_int64(0)
        self.check(lib().utv_stream_stats(self.h, C.byref(a), C.byref(b), C.byref(c)))
        return {"h2d_bytes": int(a.value), "d2h_bytes": int(b.value), "resident_cols": int(c.value)}

    # ------------------------------------------------------------------ step entry points
    def sketch(self, seed: int, step: int, row0: int, mrows: int, b: int, G=None):
        G = colmajor_empty(mrows, b, device=f"cuda:{self.device}") if G is None else G
        self.check(lib().utv_sketch(self.h, seed, step, row0, mrows, b, _ptr(G), _ld(G)))
        return G

    def philox(self, ctr: torch.Tensor, key: torch.Tensor) -> torch.Tensor:
        n = ctr.numel() // 4
        out = torch.empty(4 * n, dtype=torch.int32, device=ctr.device)
        self.check(lib().utv_philox(self.h, n, _ptr(ctr), _ptr(key), _ptr(out)))
        return out

    def hqr(self, P):
        _check_f64(P)
        m, w = P.shape
        dev = P.device
        W = colmajor_empty(m, w, device=dev)
        tau = torch.empty(w, dtype=torch.float64, device=dev)
        T = colmajor_empty(w, w, device=dev)
        self.check(lib().utv_hqr(self.h, m, w, _ptr(P), _ld(P), _ptr(W), _ld(W), _ptr(tau), _ptr(T), _ld(T)))
        return P, W, tau, T

    def svd_small(self, R):
        _check_f64(R)
        b = R.shape[0]
        dev = R.device
        Us = colmajor_empty(b, b, device=dev); Vs = colmajor_empty(b, b, device=dev)
        s = torch.empty(b, dtype=torch.float64, device=dev)
        sw = C.c_int32(0)
        self.check(lib().utv_svd_small(self.h, b, _ptr(R), _ld(R), _ptr(Us), _ld(Us), _ptr(s), _ptr(Vs), _ld(Vs),
                                       C.byref(sw)))
        return Us, s, Vs, int(sw.value)

    def svd_block(self, A11, Us=None, s=None, Vs=None):
        """A11 (b x b upper triangular, in place) := diag(sigma); returns (U_s, sigma, V_s)."""
        _check_f64(A11)
        b = A11.shape[0]
        dev = A11.device
        Us = colmajor_empty(b, b, device=dev) if Us is None else Us
        Vs = colmajor_empty(b, b, device=dev) if Vs is None else Vs
        s = torch.empty(b, dtype=torch.float64, device=dev) if s is None else s
        self.check(lib().utv_svd_block(self.h, b, _ptr(A11), _ld(A11), _ptr(Us), _ld(Us), _ptr(s), _ptr(Vs), _ld(Vs)))
        return Us, s, Vs

    def svd_status(self):
        f, sw = C.c_int32(0), C.c_int32(0)
        self.check(lib().utv_svd_status(self.h, C.byref(f), C.byref(sw)))
        return int(f.value), int(sw.value)

    def trsm_upper(self, T, Z):
        """Z := T^{-1} Z for the leading Z.shape[0] x Z.shape[0] block of upper-triangular T."""
        _check_f64(T, Z)
        n = Z.shape[0]
        k = Z.shape[1] if Z.dim() == 2 else 1
        self.check(lib().utv_trsm_upper(self.h, n, _ptr(T), _ld(T), _ptr(Z), _ld(Z), k))
        return Z

    def gemm(self, ta: bool, tb: bool, alpha: float, A, B, beta: float, Cm):
        _check_f64(A, B, Cm)
        M, N = Cm.shape
        K = A.shape[0] if ta else A.shape[1]
        self.check(lib().utv_gemm(self.h, int(ta), int(tb), M, N, K, float(alpha), _ptr(A), _ld(A), _ptr(B), _ld(B),
                                  float(beta), _ptr(Cm), _ld(Cm)))
        return Cm

    def profile(self, enable: bool):
        self.check(lib().utv_profile(self.h, int(bool(enable))))

    def profile_read(self) -> dict:
        arr = (_ProfEntry * len(PROF_FAMILIES))()
        self.check(lib().utv_profile_read(self.h, C.cast(arr, C.c_void_p)))
        return {name: {"launches": e.launches, "calls": e.calls, "ms": e.ms, "flops": e.flops, "bytes": e.bytes}
                for name, e in zip(PROF_FAMILIES, arr)}

    def profile_dump(self, path: str):
        self.check(lib().utv_profile_dump(self.h, path.encode()))

    def rank_diag(self, d, tau: float) -> int:
        r = C.c_int64(0)
        self.check(lib().utv_rank_diag(self.h, d.numel(), _ptr(d), float(tau), C.byref(r)))
        return int(r.value)

    def rank(self, T, tau: float) -> int:
        r = C.c_int64(0)
        n = T.shape[1]
        self.check(lib().utv_rank(self.h, n, _ptr(T), _ld(T), float(tau), C.byref(r)))
        return int(r.value)


_default_handles: dict = {}


def default_handle() -> Handle:
    dev = torch.cuda.current_device()
    h = _default_handles.get(dev)
    if h is None:
        h = _default_handles[dev] = Handle(dev)
    return h


def lstsq(A, B, opts: Opts | None = None, handle: Handle | None = None):
    """x_simple for min ||A x - B|| (fast option).  Consumes (overwrites) A and B.

    Returns (X, r) with X column-major (n x k) on the same device as A.
    """
    h = handle or default_handle()
    m, n = A.shape
    k = B.shape[1] if B.dim() == 2 else 1
    X = colmajor_empty(n, k, device=A.device) if A.is_cuda else colmajor_empty(n, k, device="cpu")
    r = h.lstsq(A, B if B.dim() == 2 else B.reshape(-1, 1), X, opts)
    return X, r


# ----------------------------------------------------------------------------- multi-GPU handles
def get_unique_id() -> bytes:
    """NCCL unique id (128 bytes) for dist_handle(); create it on one rank and share it."""
    buf = C.create_string_buffer(128)
    st = lib().utv_get_unique_id(buf)
    if st != UTV_OK:
        raise UtvError(st, "utv_get_unique_id failed (libnccl.so.2 unavailable?)")
    return buf.raw


def dist_handle(nccl_uid: bytes, nranks: int, rank: int, device: int | None = None) -> Handle:
    """Rank `rank` of an NCCL multi-GPU handle (one process per GPU; utv_create_dist)."""
    device = torch.cuda.current_device() if device is None else int(device)
    stream = torch.cuda.current_stream(device)
    h = C.c_void_p()
    uid = C.create_string_buffer(bytes(nccl_uid), 128)
    st = lib().utv_create_dist(C.byref(h), device, C.c_void_p(stream.cuda_stream), uid, nranks, rank)
    if st != UTV_OK:
        raise UtvError(st, "utv_create_dist failed")
    return Handle._wrap(h, device, stream)


def _cudart():
    """The CUDA runtime torch already loaded (cudaMemcpy / cudaStreamSynchronize for host staging)."""
    global _cudart_lib
    if _cudart_lib is None:
        import glob
        import os as _os
        cands = ["libcudart.so.12", "libcudart.so"]
        for d in (_os.path.join(_os.path.dirname(torch.__file__), "lib"),):
            cands += sorted(glob.glob(_os.path.join(d, "libcudart*.so*")))
        try:
            import nvidia.cuda_runtime as _ncr
            cands += sorted(glob.glob(_os.path.join(list(_ncr.__path__)[0], "lib", "libcudart.so*")))
        except Exception:
            pass
        err = None
        for c in cands:
            try:
                _cudart_lib = C.CDLL(c)
                break
            except OSError as e:
                err = e
        if _cudart_lib is None:
            raise RuntimeError(f"libcudart not found: {err}")
        _cudart_lib.cudaMemcpy.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int]
        _cudart_lib.cudaStreamSynchronize.argtypes = [C.c_void_p]
    return _cudart_lib


_cudart_lib = None


def comm_handle(rank: int, nranks: int, group=None, device: int | None = None) -> Handle:
    """Rank `rank` of a multi-GPU handle whose collectives go through torch.distributed on `group`
    (utv_create_with_comm; e.g. gloo, one process per rank).  The device buffers are staged through
    host memory in the callbacks (argument marshalling; the method's arithmetic stays in libutv)."""
    import numpy as np
    import torch.distributed as tdist
    device = torch.cuda.current_device() if device is None else int(device)
    stream = torch.cuda.current_stream(device)
    rt = _cudart()
    H2D, D2H = 1, 2

    def stage_out(buf, n, st):
        rt.cudaStreamSynchronize(C.c_void_p(st))
        a = np.empty(n, dtype=np.float64)
        if rt.cudaMemcpy(a.ctypes.data, buf, n * 8, D2H) != 0:
            raise RuntimeError("cudaMemcpy D2H failed")
        return a

    def stage_in(buf, a):
        if rt.cudaMemcpy(buf, a.ctypes.data, a.size * 8, H2D) != 0:
            raise RuntimeError("cudaMemcpy H2D failed")

    def ar(ctx, buf, n, st):
        try:
            a = stage_out(buf, n, st)
            t = torch.from_numpy(a)
            tdist.all_reduce(t, group=group)
            stage_in(buf, a)
            return 0
        except Exception:               # noqa: BLE001 -- reported to libutv as a failed collective
            return 1

    def bc(ctx, buf, n, root, st):
        try:
            a = stage_out(buf, n, st)
            t = torch.from_numpy(a)
            tdist.broadcast(t, src=tdist.get_global_rank(group, root) if group is not None else root, group=group)
            if rank != root:
                stage_in(buf, a)
            return 0
        except Exception:               # noqa: BLE001
            return 1

    def ag(ctx, send, recv, n, st):
        try:
            a = torch.from_numpy(stage_out(send, n, st))
            outs = [torch.empty(n, dtype=torch.float64) for _ in range(nranks)]
            tdist.all_gather(outs, a, group=group)
            stage_in(recv, torch.cat(outs).numpy())
            return 0
        except Exception:               # noqa: BLE001
            return 1

    def ab(ctx):
        pass

    cbs = (_AR_CB(ar), _BC_CB(bc), _AG_CB(ag), _AB_CB(ab))
    ops = _CommOps(cbs[0], cbs[1], cbs[2], cbs[3], None)
    h = C.c_void_p()
    st = lib().utv_create_with_comm(C.byref(h), device, C.c_void_p(stream.cuda_stream), nranks, rank, C.byref(ops))
    if st != UTV_OK:
        raise UtvError(st, "utv_create_with_comm failed")
    hd = Handle._wrap(h, device, stream)
    hd._callbacks = cbs                # the C function pointers must outlive the handle
    return hd


def local_group(nranks: int, devices=None, streams=None) -> list:
    """nranks handles forming one in-process multi-GPU group (utv_create_local_group); drive each
    handle from its own thread.  devices default to the current device for every rank."""
    devices = [torch.cuda.current_device()] * nranks if devices is None else list(devices)
    streams = [torch.cuda.Stream(device=d) for d in devices] if streams is None else list(streams)
    hs = (C.c_void_p * nranks)()
    devs = (C.c_int * nranks)(*devices)
    sts = (C.c_void_p * nranks)(*[s.cuda_stream for s in streams])
    st = lib().utv_create_local_group(hs, nranks, devs, sts)
    if st != UTV_OK:
        raise UtvError(st, "utv_create_local_group failed")
    return [Handle._wrap(C.c_void_p(hs[r]), devices[r], streams[r]) for r in range(nranks)]


UTV_TUNE_GEMM_CFG, UTV_TUNE_GEMM_SPLITS, UTV_TUNE_GEMM_PATH, UTV_TUNE_QR_GLOBAL, UTV_TUNE_QR_CTAS = 1, 2, 3, 4, 5
UTV_TUNE_DIST_CHUNKS, UTV_TUNE_SVD_LAG, UTV_TUNE_QR_CHOLQR = 6, 7, 8


def tune(key: int, value: int) -> int:
    """Set a process-wide implementation knob (utv_tune, include/utv_steps.h); returns the old value."""
    old = C.c_int64(0)
    st = lib().utv_tune(int(key), int(value), C.byref(old))
    if st != UTV_OK:
        raise UtvError(st, f"utv_tune: unknown key {key}")
    return int(old.value)


class tuned:
    """Context manager: ``with tuned(UTV_TUNE_GEMM_CFG, 0): ...`` forces a knob and restores it."""

    def __init__(self, *pairs):
        self.pairs = [(pairs[i], pairs[i + 1]) for i in range(0, len(pairs), 2)]
        self.old = []

    def __enter__(self):
        self.old = [(k, tune(k, v)) for k, v in self.pairs]
        return self

    def __exit__(self, *a):
        for k, v in reversed(self.old):
            tune(k, v)


def dist_local_cols(n: int, block: int, nranks: int, rank: int) -> int:
    return int(lib().utv_dist_local_cols(n, block, nranks, rank))
