"""Python binding of libtf.so — the B200 (sm_100a) dGN evaluation hot path of Tensor Fox.

Argument marshalling only: every function here validates shapes/dtypes, takes the
device pointers of torch tensors (PyTorch supplies memory and streams) and calls
the C ABI of include/tf.h with the same names. All arithmetic of the method runs
in the CUDA kernels behind that ABI. There is no CPU fallback: importing this
package raises if libtf.so is missing, and every call raises on a non-OK status.

Layouts (include/tf.h): T is a contiguous fp64 tensor of shape (K, J, I) — i.e.
first index fastest, T[i + I*(j + J*k)] — or any tensor whose memory is that;
w = [vec A; vec B; vec C] (column-major factors), length n = R*(I+J+K_total).
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TF_LIB_PATH") or os.path.join(_HERE, "libtf.so")   # TF_LIB_PATH: dev builds only

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python paper_2110_05997_b200/build.py` "
        "(nvcc, sm_100a). There is no CPU fallback.")

_lib = ctypes.CDLL(LIB_PATH)


class TfDims(ctypes.Structure):
    _fields_ = [("I", ctypes.c_int64), ("J", ctypes.c_int64), ("K", ctypes.c_int64), ("R", ctypes.c_int64),
                ("ldT", ctypes.c_int64), ("K_total", ctypes.c_int64), ("k_begin", ctypes.c_int64)]


_vp = ctypes.c_void_p
ALLREDUCE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.POINTER(ctypes.c_double), ctypes.c_int64, ctypes.c_void_p)
_lib.tf_ctx_create.argtypes = [ctypes.POINTER(_vp), ctypes.c_int, _vp]
_lib.tf_ctx_destroy.argtypes = [_vp]
_lib.tf_ctx_set_stream.argtypes = [_vp, _vp]
_lib.tf_status_str.restype = ctypes.c_char_p
_lib.tf_status_str.argtypes = [ctypes.c_int]
_lib.tf_last_error.restype = ctypes.c_char_p
_lib.tf_last_error.argtypes = [_vp]
_lib.tf_grams.argtypes = [_vp, TfDims, _vp, _vp]
_lib.tf_hadamard.argtypes = [_vp, ctypes.c_int64, _vp, _vp]
_lib.tf_cpd_eval.argtypes = [_vp, TfDims, _vp, _vp, _vp, _vp, _vp]
_lib.tf_cpd_eval_host.argtypes = [_vp, TfDims, _vp, _vp, _vp, _vp]
_lib.tf_gn_matvec.argtypes = [_vp, TfDims, _vp, _vp, _vp, ctypes.c_double, _vp]
_lib.tf_cg_solve.argtypes = [_vp, TfDims, _vp, _vp, _vp, ctypes.c_double, ctypes.c_int, ctypes.c_double,
                             ctypes.c_int, _vp, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_double)]
_lib.tf_reg_gamma.argtypes = [_vp, ctypes.c_int64, _vp, _vp]
_lib.tf_gn_matvec_damped.argtypes = [_vp, TfDims, _vp, _vp, _vp, ctypes.c_double, _vp, _vp]
_lib.tf_cg_solve_damped.argtypes = [_vp, TfDims, _vp, _vp, _vp, ctypes.c_double, _vp, ctypes.c_int, ctypes.c_double,
                                    ctypes.c_int, _vp, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_double)]
class TfDgnParams(ctypes.Structure):
    _fields_ = [("maxiter", ctypes.c_int), ("tol", ctypes.c_double), ("mu0", ctypes.c_double),
                ("use_gamma", ctypes.c_int), ("jacobi", ctypes.c_int), ("balance", ctypes.c_int),
                ("cg_iters", ctypes.POINTER(ctypes.c_int))]


class TfDgnResult(ctypes.Structure):
    _fields_ = [("iters", ctypes.c_int), ("reason", ctypes.c_int), ("f", ctypes.c_double),
                ("rel_err", ctypes.c_double), ("mu", ctypes.c_double)]


_lib.tf_cpd_dgn.argtypes = [_vp, TfDims, _vp, _vp, ctypes.POINTER(TfDgnParams), ctypes.POINTER(TfDgnResult),
                            ctypes.POINTER(ctypes.c_double)]
_lib.tf_ctx_set_timing.argtypes = [_vp, ctypes.c_int]
_lib.tf_ctx_set_eval_form.argtypes = [_vp, ctypes.c_int]
_lib.tf_ctx_set_cg_grid.argtypes = [_vp, ctypes.c_int]
_lib.tf_ctx_eval_path.argtypes = [_vp, ctypes.POINTER(ctypes.c_int)]
_lib.tf_cpd_dgn_sharded.argtypes = [_vp, TfDims, _vp, _vp, ctypes.POINTER(TfDgnParams), ctypes.POINTER(TfDgnResult),
                                    ctypes.POINTER(ctypes.c_double), ALLREDUCE_FN, ctypes.c_void_p, _vp]
_lib.tf_ctx_eval_fallback.argtypes = [_vp, ctypes.POINTER(ctypes.c_int)]
_i64 = ctypes.c_int64
_lib.tf_unfolding_grams.argtypes = [_vp, TfDims, _vp, _vp, _vp, _vp]
_lib.tf_sym_eig_top.argtypes = [_vp, _i64, _vp, _i64, _vp, ctypes.c_int, ctypes.c_double, _vp, _vp,
                                ctypes.POINTER(ctypes.c_int)]
_lib.tf_multilinear_core.argtypes = [_vp, TfDims, _vp, _vp, _i64, _vp, _i64, _vp, _i64, _vp]
_lib.tf_compress.argtypes = [_vp, TfDims, _vp, _vp, ctypes.c_double, ctypes.c_int, ctypes.c_double, _vp, _vp, _vp,
                             ctypes.POINTER(_i64), ctypes.POINTER(ctypes.c_int)]
_lib.tf_compress_st.argtypes = [_vp, TfDims, _vp, _vp, ctypes.c_double, ctypes.c_int, ctypes.c_double, _vp, _vp,
                                _vp, ctypes.POINTER(_i64), ctypes.POINTER(ctypes.c_int)]
_lib.tf_compress_st_sharded.argtypes = [_vp, TfDims, _vp, _vp, ctypes.c_double, ctypes.c_int, ctypes.c_double, _vp,
                                        _vp, _vp, ctypes.POINTER(_i64), ctypes.POINTER(ctypes.c_int), ALLREDUCE_FN,
                                        ctypes.c_void_p, _vp]
_lib.tf_energy_init.argtypes = [_vp, _i64, _i64, _i64, _vp, _i64, _vp]
_lib.tf_uncompress.argtypes = [_vp, _i64, _i64, _vp, _vp, _i64, _vp]


_lib.tf_mttkrp.argtypes = [_vp, TfDims, _vp, _vp, ctypes.c_int, _vp]
_lib.tf_als.argtypes = [_vp, TfDims, _vp, _vp, ctypes.c_int, ctypes.POINTER(ctypes.c_double)]


class TfCpdParams(ctypes.Structure):
    _fields_ = [("mlsvd_tol", ctypes.c_double), ("eig_maxiter", ctypes.c_int), ("init", ctypes.c_int),
                ("dgn", TfDgnParams), ("sequential", ctypes.c_int)]


class TfCpdResult(ctypes.Structure):
    _fields_ = [("ranks", _i64 * 3), ("eig_iters", ctypes.c_int * 3), ("dgn", TfDgnResult),
                ("rel_err", ctypes.c_double)]


_lib.tf_cpd.argtypes = [_vp, TfDims, _vp, _vp, _vp, ctypes.POINTER(TfCpdParams), _vp, _vp, ctypes.POINTER(TfCpdResult),
                        ctypes.POINTER(ctypes.c_double)]
_lib.tf_cpd_sharded.argtypes = [_vp, TfDims, _vp, _vp, _vp, ctypes.POINTER(TfCpdParams), _vp, _vp,
                                ctypes.POINTER(TfCpdResult), ctypes.POINTER(ctypes.c_double), ALLREDUCE_FN,
                                ctypes.c_void_p, _vp]
_lib.tf_ctx_kernel_stats.argtypes = [_vp, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int64),
                                     ctypes.POINTER(ctypes.c_int64), ctypes.c_int]

EXPORTED = ["tf_ctx_create", "tf_ctx_destroy", "tf_ctx_set_stream", "tf_status_str", "tf_last_error", "tf_version",
            "tf_grams", "tf_hadamard", "tf_cpd_eval", "tf_cpd_eval_host", "tf_gn_matvec", "tf_cg_solve",
            "tf_reg_gamma", "tf_gn_matvec_damped", "tf_cg_solve_damped", "tf_cpd_dgn", "tf_ctx_set_timing",
            "tf_ctx_kernel_stats", "tf_unfolding_grams", "tf_sym_eig_top", "tf_multilinear_core", "tf_compress",
            "tf_energy_init", "tf_uncompress", "tf_cpd", "tf_mttkrp", "tf_als", "tf_ctx_set_eval_form", "tf_ctx_set_cg_grid", "tf_ctx_eval_path",
            "tf_ctx_eval_fallback", "tf_cpd_dgn_sharded", "tf_compress_st",
            "tf_compress_st_sharded", "tf_cpd_sharded"]

TF_OK, TF_ERR_ARG, TF_ERR_ALIGN, TF_ERR_UNSUPPORTED, TF_ERR_CUDA, TF_ERR_NONFINITE, TF_ERR_ALLOC = range(7)
MAX_R = 128


class TfError(RuntimeError):
    def __init__(self, status: int, detail: str):
        self.status = status
        super().__init__(f"{_lib.tf_status_str(status).decode()}: {detail}")


@dataclass
class Dims:
    I: int
    J: int
    K: int
    R: int
    ldT: int = 0
    K_total: int = 0
    k_begin: int = 0

    def c(self) -> TfDims:
        return TfDims(self.I, self.J, self.K, self.R, self.ldT, self.K_total, self.k_begin)

    @property
    def Kt(self) -> int:
        return self.K_total or (self.K + self.k_begin)

    @property
    def n(self) -> int:
        return self.R * (self.I + self.J + self.Kt)


def _ptr(t: torch.Tensor | None):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _dev(t: torch.Tensor, name: str, numel: int | None = None):
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor")
    if t.dtype != torch.float64:
        raise TypeError(f"{name} must be float64")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if numel is not None and t.numel() < numel:
        raise ValueError(f"{name} has {t.numel()} elements, needs {numel}")


def _make_hook(xbuf: torch.Tensor, allreduce):
    """A C all-reduce hook (tf_allreduce_fn) that SUM-reduces the first `count` doubles of the torch tensor
    xbuf (the exchange buffer the library was given) with the Python callable allreduce(view); exceptions
    are kept (never raised across the C ABI) and re-raised by the caller."""
    errors = []

    def hook(buf, count, user):
        try:
            allreduce(xbuf[:count])
            torch.cuda.current_stream(xbuf.device).synchronize()
            return 0
        except Exception as e:
            errors.append(e)
            return 1

    return ALLREDUCE_FN(hook), errors


class Context:
    """A tf_ctx bound to one device and a CUDA stream (default: torch's current stream)."""

    def __init__(self, device: int | torch.device | None = None, stream: torch.cuda.Stream | None = None):
        if device is None:
            device = torch.cuda.current_device()
        if isinstance(device, torch.device):
            device = device.index if device.index is not None else torch.cuda.current_device()
        self.device = int(device)
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        h = _vp()
        st = _lib.tf_ctx_create(ctypes.byref(h), self.device, _vp(self.stream.cuda_stream))
        if st != TF_OK:
            raise TfError(st, "tf_ctx_create failed")
        self._h = h

    def _check(self, st: int):
        if st != TF_OK:
            raise TfError(st, _lib.tf_last_error(self._h).decode())

    def set_stream(self, stream: torch.cuda.Stream):
        self.stream = stream
        self._check(_lib.tf_ctx_set_stream(self._h, _vp(stream.cuda_stream)))

    def close(self):
        if getattr(self, "_h", None):
            _lib.tf_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------------ the C-ABI calls
    def tf_grams(self, d: Dims, w: torch.Tensor, grams: torch.Tensor | None = None) -> torch.Tensor:
        _dev(w, "w", d.n)
        if grams is None:
            grams = torch.empty(3 * d.R * d.R, dtype=torch.float64, device=w.device)
        _dev(grams, "grams", 3 * d.R * d.R)
        self._check(_lib.tf_grams(self._h, d.c(), _ptr(w), _ptr(grams)))
        return grams

    def tf_hadamard(self, R: int, grams: torch.Tensor, pi: torch.Tensor | None = None) -> torch.Tensor:
        _dev(grams, "grams", 3 * R * R)
        if pi is None:
            pi = torch.empty(6 * R * R, dtype=torch.float64, device=grams.device)
        _dev(pi, "pi", 6 * R * R)
        self._check(_lib.tf_hadamard(self._h, R, _ptr(grams), _ptr(pi)))
        return pi

    def tf_cpd_eval(self, d: Dims, T: torch.Tensor, w: torch.Tensor, f: torch.Tensor | None = None,
                    grad: torch.Tensor | None = None, grams: torch.Tensor | None = None):
        """Returns (f, grad) device tensors (f has one element)."""
        ldT = d.ldT or d.I
        _dev(T, "T", ldT * d.J * d.K - (ldT - d.I))
        _dev(w, "w", d.n)
        if f is None:
            f = torch.empty(1, dtype=torch.float64, device=w.device)
        if grad is None:
            grad = torch.empty(d.n, dtype=torch.float64, device=w.device)
        _dev(f, "f", 1)
        _dev(grad, "grad", d.n)
        if grams is not None:
            _dev(grams, "grams", 3 * d.R * d.R)
        self._check(_lib.tf_cpd_eval(self._h, d.c(), _ptr(T), _ptr(w), _ptr(f), _ptr(grad), _ptr(grams)))
        return f, grad

    def tf_cpd_eval_host(self, d: Dims, T_host: torch.Tensor, w_host: torch.Tensor,
                         f_host: torch.Tensor | None = None, grad_host: torch.Tensor | None = None):
        """Host-buffer evaluation: T streamed to the device in slabs (synchronizes)."""
        for name, t in (("T_host", T_host), ("w_host", w_host)):
            if t.is_cuda or t.dtype != torch.float64 or not t.is_contiguous():
                raise TypeError(f"{name} must be a contiguous float64 CPU tensor")
        if f_host is None:
            f_host = torch.empty(1, dtype=torch.float64)
        if grad_host is None:
            grad_host = torch.empty(d.n, dtype=torch.float64)
        self._check(_lib.tf_cpd_eval_host(self._h, d.c(), _ptr(T_host), _ptr(w_host), _ptr(f_host),
                                          _ptr(grad_host)))
        return f_host, grad_host

    def tf_gn_matvec(self, d: Dims, grams: torch.Tensor, w: torch.Tensor, v: torch.Tensor, lam: float,
                     y: torch.Tensor | None = None) -> torch.Tensor:
        _dev(grams, "grams", 3 * d.R * d.R)
        _dev(w, "w", d.n)
        _dev(v, "v", d.n)
        if y is None:
            y = torch.empty(d.n, dtype=torch.float64, device=w.device)
        _dev(y, "y", d.n)
        self._check(_lib.tf_gn_matvec(self._h, d.c(), _ptr(grams), _ptr(w), _ptr(v), float(lam), _ptr(y)))
        return y

    def tf_cg_solve(self, d: Dims, grams: torch.Tensor, w: torch.Tensor, rhs: torch.Tensor, lam: float,
                    maxiter: int, tol: float = 0.0, jacobi: bool = False, x: torch.Tensor | None = None):
        """Returns (x, iters_done, ||r||^2)."""
        _dev(grams, "grams", 3 * d.R * d.R)
        _dev(w, "w", d.n)
        _dev(rhs, "rhs", d.n)
        if x is None:
            x = torch.empty(d.n, dtype=torch.float64, device=w.device)
        _dev(x, "x", d.n)
        it = ctypes.c_int()
        r2 = ctypes.c_double()
        self._check(_lib.tf_cg_solve(self._h, d.c(), _ptr(grams), _ptr(w), _ptr(rhs), float(lam), int(maxiter),
                                     float(tol), int(bool(jacobi)), _ptr(x), ctypes.byref(it), ctypes.byref(r2)))
        return x, it.value, r2.value

    def tf_reg_gamma(self, R: int, grams: torch.Tensor, gamma: torch.Tensor | None = None) -> torch.Tensor:
        """Tensor Fox's diagonal regularizer gamma (3R) from the Grams."""
        _dev(grams, "grams", 3 * R * R)
        if gamma is None:
            gamma = torch.empty(3 * R, dtype=torch.float64, device=grams.device)
        _dev(gamma, "gamma", 3 * R)
        self._check(_lib.tf_reg_gamma(self._h, R, _ptr(grams), _ptr(gamma)))
        return gamma

    def tf_gn_matvec_damped(self, d: Dims, grams: torch.Tensor, w: torch.Tensor, v: torch.Tensor, mu: float,
                            damp: torch.Tensor | None, y: torch.Tensor | None = None) -> torch.Tensor:
        _dev(grams, "grams", 3 * d.R * d.R)
        _dev(w, "w", d.n)
        _dev(v, "v", d.n)
        if damp is not None:
            _dev(damp, "damp", 3 * d.R)
        if y is None:
            y = torch.empty(d.n, dtype=torch.float64, device=w.device)
        _dev(y, "y", d.n)
        self._check(_lib.tf_gn_matvec_damped(self._h, d.c(), _ptr(grams), _ptr(w), _ptr(v), float(mu), _ptr(damp),
                                             _ptr(y)))
        return y

    def tf_cg_solve_damped(self, d: Dims, grams: torch.Tensor, w: torch.Tensor, rhs: torch.Tensor, mu: float,
                           damp: torch.Tensor | None, maxiter: int, tol: float = 0.0, jacobi: bool = False,
                           x: torch.Tensor | None = None):
        """Returns (x, iters_done, ||r||^2) for (J^T J + mu D) x = rhs."""
        _dev(grams, "grams", 3 * d.R * d.R)
        _dev(w, "w", d.n)
        _dev(rhs, "rhs", d.n)
        if damp is not None:
            _dev(damp, "damp", 3 * d.R)
        if x is None:
            x = torch.empty(d.n, dtype=torch.float64, device=w.device)
        _dev(x, "x", d.n)
        it = ctypes.c_int()
        r2 = ctypes.c_double()
        self._check(_lib.tf_cg_solve_damped(self._h, d.c(), _ptr(grams), _ptr(w), _ptr(rhs), float(mu), _ptr(damp),
                                            int(maxiter), float(tol), int(bool(jacobi)), _ptr(x), ctypes.byref(it),
                                            ctypes.byref(r2)))
        return x, it.value, r2.value

    # ------------------------------------------------------------------ compression stage (NEXT #3)
    def tf_unfolding_grams(self, d: Dims, T: torch.Tensor, modes=(1, 2, 3)):
        """[G1, G2, G3] = T_(l) T_(l)^T (None for modes not requested); each (I_l, I_l), column-major
        storage, symmetric."""
        ldT = d.ldT or d.I
        _dev(T, "T", ldT * d.J * d.K - (ldT - d.I))
        dims = (d.I, d.J, d.K)
        out = [torch.empty(dims[l] * dims[l], dtype=torch.float64, device=T.device) if (l + 1) in modes else None
               for l in range(3)]
        self._check(_lib.tf_unfolding_grams(self._h, d.c(), _ptr(T), _ptr(out[0]), _ptr(out[1]), _ptr(out[2])))
        return out

    def tf_sym_eig_top(self, n: int, G: torch.Tensor, P: int, Omega: torch.Tensor, maxiter: int = 100,
                       tol: float = 0.0):
        """(U (n*P, column-major), lam (P,), iterations) — top-P eigenpairs of the symmetric PSD G."""
        _dev(G, "G", n * n)
        _dev(Omega, "Omega", n * P)
        U = torch.empty(n * P, dtype=torch.float64, device=G.device)
        lam = torch.empty(P, dtype=torch.float64, device=G.device)
        it = ctypes.c_int()
        self._check(_lib.tf_sym_eig_top(self._h, n, _ptr(G), P, _ptr(Omega), int(maxiter), float(tol), _ptr(U),
                                        _ptr(lam), ctypes.byref(it)))
        return U, lam, it.value

    def tf_multilinear_core(self, d: Dims, T: torch.Tensor, U1, P1: int, U2, P2: int, U3, P3: int):
        """S = (U1^T, U2^T, U3^T)·T as a flat (P1*P2*P3,) first-index-fastest tensor."""
        ldT = d.ldT or d.I
        _dev(T, "T", ldT * d.J * d.K - (ldT - d.I))
        for name, U, n, P in (("U1", U1, d.I, P1), ("U2", U2, d.J, P2), ("U3", U3, d.K, P3)):
            _dev(U, name, n * P)
        S = torch.empty(P1 * P2 * P3, dtype=torch.float64, device=T.device)
        self._check(_lib.tf_multilinear_core(self._h, d.c(), _ptr(T), _ptr(U1), P1, _ptr(U2), P2, _ptr(U3), P3,
                                             _ptr(S)))
        return S

    def tf_compress(self, d: Dims, T: torch.Tensor, Omega: torch.Tensor, mlsvd_tol: float = 1e-6,
                    eig_maxiter: int = 100, eig_tol: float = 0.0, sequential: bool = False):
        """Alg. Compression (sequential=True: Alg. ST-MLSVD). Returns dict(U=[U1, U2, U3] (I_l x P_l,
        column-major flat), sigma=[...],
        S=core (R~1*R~2*R~3,), ranks=(R~1, R~2, R~3), P=(P1, P2, P3), eig_iters=[...])."""
        ldT = d.ldT or d.I
        _dev(T, "T", ldT * d.J * d.K - (ldT - d.I))
        dims = (d.I, d.J, d.K)
        P = tuple(min(n, d.R) for n in dims)
        nU = sum(n * p for n, p in zip(dims, P))
        _dev(Omega, "Omega", nU)
        U = torch.empty(nU, dtype=torch.float64, device=T.device)
        sigma = torch.empty(sum(P), dtype=torch.float64, device=T.device)
        S = torch.empty(P[0] * P[1] * P[2], dtype=torch.float64, device=T.device)
        ranks = (ctypes.c_int64 * 3)()
        iters = (ctypes.c_int * 3)()
        fn = _lib.tf_compress_st if sequential else _lib.tf_compress
        self._check(fn(self._h, d.c(), _ptr(T), _ptr(Omega), float(mlsvd_tol), int(eig_maxiter),
                       float(eig_tol), _ptr(U), _ptr(sigma), _ptr(S), ranks, iters))
        rk = tuple(int(r) for r in ranks)
        offs = [0, dims[0] * P[0], dims[0] * P[0] + dims[1] * P[1]]
        soffs = [0, P[0], P[0] + P[1]]
        return {"U": [U[offs[l]:offs[l] + dims[l] * P[l]] for l in range(3)],
                "sigma": [sigma[soffs[l]:soffs[l] + P[l]] for l in range(3)],
                "S": S[:rk[0] * rk[1] * rk[2]], "ranks": rk, "P": P, "eig_iters": [int(i) for i in iters]}

    def tf_compress_st(self, d: Dims, T: torch.Tensor, Omega: torch.Tensor, mlsvd_tol: float = 1e-6,
                       eig_maxiter: int = 100, eig_tol: float = 0.0):
        """Alg. ST-MLSVD (the sequentially truncated compression); same outputs as tf_compress."""
        return self.tf_compress(d, T, Omega, mlsvd_tol, eig_maxiter, eig_tol, sequential=True)

    def tf_compress_st_sharded(self, d: Dims, T_local: torch.Tensor, Omega: torch.Tensor, allreduce,
                               mlsvd_tol: float = 1e-6, eig_maxiter: int = 100, eig_tol: float = 0.0):
        """K-sharded Alg. ST-MLSVD (this rank: d.K slices from d.k_begin of d.K_total). allreduce(buf) must SUM
        the float64 CUDA tensor buf over the ranks in place. Same outputs as tf_compress (identical on every
        rank; U3 has K_total rows)."""
        ldT = d.ldT or d.I
        _dev(T_local, "T_local", ldT * d.J * d.K - (ldT - d.I))
        dims = (d.I, d.J, d.Kt)
        P = tuple(min(n, d.R) for n in dims)
        nU = sum(n * p for n, p in zip(dims, P))
        _dev(Omega, "Omega", nU)
        U = torch.empty(nU, dtype=torch.float64, device=T_local.device)
        sigma = torch.empty(sum(P), dtype=torch.float64, device=T_local.device)
        S = torch.empty(P[0] * P[1] * P[2], dtype=torch.float64, device=T_local.device)
        ranks = (ctypes.c_int64 * 3)()
        iters = (ctypes.c_int * 3)()
        xbuf = torch.empty(max(d.I * d.I, d.J * d.J, P[0] * P[1] * d.Kt, 3), dtype=torch.float64,
                           device=T_local.device)
        cb, errors = _make_hook(xbuf, allreduce)
        st = _lib.tf_compress_st_sharded(self._h, d.c(), _ptr(T_local), _ptr(Omega), float(mlsvd_tol),
                                         int(eig_maxiter), float(eig_tol), _ptr(U), _ptr(sigma), _ptr(S), ranks, iters,
                                         cb, None, _ptr(xbuf))
        if errors:
            raise errors[0]
        self._check(st)
        rk = tuple(int(r) for r in ranks)
        offs = [0, dims[0] * P[0], dims[0] * P[0] + dims[1] * P[1]]
        soffs = [0, P[0], P[0] + P[1]]
        return {"U": [U[offs[l]:offs[l] + dims[l] * P[l]] for l in range(3)],
                "sigma": [sigma[soffs[l]:soffs[l] + P[l]] for l in range(3)],
                "S": S[:rk[0] * rk[1] * rk[2]], "ranks": rk, "P": P, "eig_iters": [int(i) for i in iters]}

    def tf_energy_init(self, R1: int, R2: int, R3: int, S: torch.Tensor, R: int) -> torch.Tensor:
        """Packed w = [vec W1; vec W2; vec W3] of the MLSVD-energy initialisation on the core S."""
        _dev(S, "S", R1 * R2 * R3)
        w = torch.empty(R * (R1 + R2 + R3), dtype=torch.float64, device=S.device)
        self._check(_lib.tf_energy_init(self._h, R1, R2, R3, _ptr(S), R, _ptr(w)))
        return w

    def tf_uncompress(self, n: int, Rl: int, U: torch.Tensor, W: torch.Tensor, R: int) -> torch.Tensor:
        """out (n x R, column-major flat) = U (n x Rl) W (Rl x R)."""
        _dev(U, "U", n * Rl)
        _dev(W, "W", Rl * R)
        out = torch.empty(n * R, dtype=torch.float64, device=U.device)
        self._check(_lib.tf_uncompress(self._h, n, Rl, _ptr(U), _ptr(W), R, _ptr(out)))
        return out

    def tf_cpd_dgn(self, d: Dims, T: torch.Tensor, w: torch.Tensor, cg_iters, maxiter: int | None = None,
                   tol: float = 1e-6, mu0: float = 0.0, use_gamma: bool = True, jacobi: bool = True,
                   balance: bool = True):
        """Tensor Fox's dGN loop on the device; w (device) is updated in place.
        cg_iters: the per-iteration random CG budgets (e.g. synth.cg_budget). Returns (result dict, history
        array [iters, 5] = F, rel_err, mu, g, ||x||)."""
        import numpy as np
        ldT = d.ldT or d.I
        _dev(T, "T", ldT * d.J * d.K - (ldT - d.I))
        _dev(w, "w", d.n)
        cgi = np.ascontiguousarray(np.asarray(cg_iters, dtype=np.int32))
        m = int(maxiter if maxiter is not None else cgi.size)
        if cgi.size < m:
            raise ValueError("cg_iters shorter than maxiter")
        prm = TfDgnParams(m, float(tol), float(mu0), int(bool(use_gamma)), int(bool(jacobi)), int(bool(balance)),
                          cgi.ctypes.data_as(ctypes.POINTER(ctypes.c_int)))
        res = TfDgnResult()
        hist = np.zeros(5 * max(m, 1))
        self._check(_lib.tf_cpd_dgn(self._h, d.c(), _ptr(T), _ptr(w), ctypes.byref(prm), ctypes.byref(res),
                                    hist.ctypes.data_as(ctypes.POINTER(ctypes.c_double))))
        out = {"iters": res.iters, "reason": res.reason, "f": res.f, "rel_err": res.rel_err, "mu": res.mu}
        return out, hist.reshape(-1, 5)[:res.iters]

    def tf_cpd(self, d: Dims, T: torch.Tensor, Omega: torch.Tensor, cg_iters, w0_core: torch.Tensor | None = None,
               mlsvd_tol: float = 1e-6, eig_maxiter: int = 100, maxiter: int | None = None, tol: float = 1e-6,
               mu0: float = 0.0, use_gamma: bool = True, jacobi: bool = True, balance: bool = True,
               sequential: bool = False):
        """The whole Tensor Fox flow: compression (sequential=True: Alg. ST-MLSVD), initialisation (MLSVD energy when w0_core is None, else
        the given [W1 | W2 | W3] random start on the P_l-row blocks), dGN on the core, uncompression and the
        unit-column output. Returns (W (n,), lambda (R,), result dict, dGN history on the core)."""
        import numpy as np
        ldT = d.ldT or d.I
        _dev(T, "T", ldT * d.J * d.K - (ldT - d.I))
        dims = (d.I, d.J, d.K)
        P = [min(x, d.R) for x in dims]
        _dev(Omega, "Omega", sum(x * p for x, p in zip(dims, P)))
        if w0_core is not None:
            _dev(w0_core, "w0_core", d.R * sum(P))
        cgi = np.ascontiguousarray(np.asarray(cg_iters, dtype=np.int32))
        m = int(maxiter if maxiter is not None else cgi.size)
        if cgi.size < m:
            raise ValueError("cg_iters shorter than maxiter")
        dp = TfDgnParams(m, float(tol), float(mu0), int(bool(use_gamma)), int(bool(jacobi)), int(bool(balance)),
                         cgi.ctypes.data_as(ctypes.POINTER(ctypes.c_int)))
        prm = TfCpdParams(float(mlsvd_tol), int(eig_maxiter), 0 if w0_core is not None else 1, dp, int(bool(sequential)))
        res = TfCpdResult()
        W = torch.empty(d.R * sum(dims), dtype=torch.float64, device=T.device)
        lam = torch.empty(d.R, dtype=torch.float64, device=T.device)
        hist = np.zeros(5 * max(m, 1))
        self._check(_lib.tf_cpd(self._h, d.c(), _ptr(T), _ptr(Omega), _ptr(w0_core), ctypes.byref(prm), _ptr(W),
                                _ptr(lam), ctypes.byref(res), hist.ctypes.data_as(ctypes.POINTER(ctypes.c_double))))
        out = {"ranks": tuple(int(x) for x in res.ranks), "eig_iters": [int(x) for x in res.eig_iters],
               "dgn": {"iters": res.dgn.iters, "reason": res.dgn.reason, "f": res.dgn.f, "rel_err": res.dgn.rel_err,
                       "mu": res.dgn.mu}, "rel_err": res.rel_err}
        return W, lam, out, hist.reshape(-1, 5)[:res.dgn.iters]

    # ------------------------------------------------------------------ CP-ALS (NEXT #4)
    def tf_mttkrp(self, d: Dims, T: torch.Tensor, w: torch.Tensor, mode: int, M: torch.Tensor | None = None):
        """M = T_(mode) (⊙ of the other factors), (I_mode x R) column-major flat."""
        ldT = d.ldT or d.I
        _dev(T, "T", ldT * d.J * d.K - (ldT - d.I))
        _dev(w, "w", d.n)
        rows = (d.I, d.J, d.K)[mode - 1] if mode in (1, 2, 3) else 1   # a bad mode is the library's TF_ERR_ARG
        if M is None:
            M = torch.empty(rows * d.R, dtype=torch.float64, device=T.device)
        _dev(M, "M", rows * d.R)
        self._check(_lib.tf_mttkrp(self._h, d.c(), _ptr(T), _ptr(w), int(mode), _ptr(M)))
        return M

    def tf_als(self, d: Dims, T: torch.Tensor, w: torch.Tensor, sweeps: int, track_f: bool = False):
        """Alg. ALS sweeps on w (device, in place). Returns F after every update (3*sweeps) if track_f."""
        import numpy as np
        ldT = d.ldT or d.I
        _dev(T, "T", ldT * d.J * d.K - (ldT - d.I))
        _dev(w, "w", d.n)
        fh = np.zeros(max(3 * sweeps, 1)) if track_f else None
        self._check(_lib.tf_als(self._h, d.c(), _ptr(T), _ptr(w), int(sweeps),
                                fh.ctypes.data_as(ctypes.POINTER(ctypes.c_double)) if track_f else None))
        return fh[:3 * sweeps] if track_f else None

    def tf_cpd_dgn_sharded(self, d: Dims, T_local: torch.Tensor, w: torch.Tensor, cg_iters, allreduce,
                           maxiter: int | None = None, tol: float = 1e-6, mu0: float = 0.0, use_gamma: bool = True,
                           jacobi: bool = True, balance: bool = True):
        """The dGN loop on this rank's K-shard (d.K local slices starting at d.k_begin of d.K_total).
        allreduce(buf) must replace the float64 CUDA tensor `buf` by its elementwise SUM over the ranks, in
        place (e.g. torch.distributed.all_reduce); it is called with the library's stream synchronized.
        Returns (result dict, history) like tf_cpd_dgn; w (full, replicated) is updated in place."""
        import numpy as np
        ldT = d.ldT or d.I
        _dev(T_local, "T_local", ldT * d.J * d.K - (ldT - d.I))
        _dev(w, "w", d.n)
        cgi = np.ascontiguousarray(np.asarray(cg_iters, dtype=np.int32))
        m = int(maxiter if maxiter is not None else cgi.size)
        if cgi.size < m:
            raise ValueError("cg_iters shorter than maxiter")
        prm = TfDgnParams(m, float(tol), float(mu0), int(bool(use_gamma)), int(bool(jacobi)), int(bool(balance)),
                          cgi.ctypes.data_as(ctypes.POINTER(ctypes.c_int)))
        res = TfDgnResult()
        hist = np.zeros(5 * max(m, 1))
        xbuf = torch.empty(d.n + 1, dtype=torch.float64, device=w.device)
        cb, errors = _make_hook(xbuf, allreduce)
        st = _lib.tf_cpd_dgn_sharded(self._h, d.c(), _ptr(T_local), _ptr(w), ctypes.byref(prm), ctypes.byref(res),
                                     hist.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), cb, None, _ptr(xbuf))
        if errors:
            raise errors[0]
        self._check(st)
        out = {"iters": res.iters, "reason": res.reason, "f": res.f, "rel_err": res.rel_err, "mu": res.mu}
        return out, hist.reshape(-1, 5)[:res.iters]

    def tf_cpd_sharded(self, d: Dims, T_local: torch.Tensor, Omega: torch.Tensor, cg_iters, allreduce,
                       w0_core: torch.Tensor | None = None, mlsvd_tol: float = 1e-6, eig_maxiter: int = 100,
                       maxiter: int | None = None, tol: float = 1e-6, mu0: float = 0.0, use_gamma: bool = True,
                       jacobi: bool = True, balance: bool = True):
        """The whole flow on a K-sharded tensor (always ST-MLSVD compression); returns what tf_cpd returns,
        identical on every rank."""
        import numpy as np
        ldT = d.ldT or d.I
        _dev(T_local, "T_local", ldT * d.J * d.K - (ldT - d.I))
        dims = (d.I, d.J, d.Kt)
        P = [min(x, d.R) for x in dims]
        _dev(Omega, "Omega", sum(x * p for x, p in zip(dims, P)))
        if w0_core is not None:
            _dev(w0_core, "w0_core", d.R * sum(P))
        cgi = np.ascontiguousarray(np.asarray(cg_iters, dtype=np.int32))
        m = int(maxiter if maxiter is not None else cgi.size)
        if cgi.size < m:
            raise ValueError("cg_iters shorter than maxiter")
        dp = TfDgnParams(m, float(tol), float(mu0), int(bool(use_gamma)), int(bool(jacobi)), int(bool(balance)),
                         cgi.ctypes.data_as(ctypes.POINTER(ctypes.c_int)))
        prm = TfCpdParams(float(mlsvd_tol), int(eig_maxiter), 0 if w0_core is not None else 1, dp, 1)
        res = TfCpdResult()
        W = torch.empty(d.R * sum(dims), dtype=torch.float64, device=T_local.device)
        lam = torch.empty(d.R, dtype=torch.float64, device=T_local.device)
        hist = np.zeros(5 * max(m, 1))
        xbuf = torch.empty(max(d.I * d.I, d.J * d.J, P[0] * P[1] * d.Kt, 3), dtype=torch.float64,
                           device=T_local.device)
        cb, errors = _make_hook(xbuf, allreduce)
        st = _lib.tf_cpd_sharded(self._h, d.c(), _ptr(T_local), _ptr(Omega), _ptr(w0_core), ctypes.byref(prm),
                                 _ptr(W), _ptr(lam), ctypes.byref(res),
                                 hist.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), cb, None, _ptr(xbuf))
        if errors:
            raise errors[0]
        self._check(st)
        out = {"ranks": tuple(int(x) for x in res.ranks), "eig_iters": [int(x) for x in res.eig_iters],
               "dgn": {"iters": res.dgn.iters, "reason": res.dgn.reason, "f": res.dgn.f, "rel_err": res.dgn.rel_err,
                       "mu": res.dgn.mu}, "rel_err": res.rel_err}
        return W, lam, out, hist.reshape(-1, 5)[:res.dgn.iters]

    def set_eval_form(self, form: str):
        """'auto' (default: the guarded Pi form, 4IJKR flops, when large enough), 'pi' (guarded Pi form at any
        size) or 'residual' (6IJKR flops) for tf_cpd_eval."""
        self._check(_lib.tf_ctx_set_eval_form(self._h, {"auto": 0, "residual": 1, "pi": 2}[form]))

    def eval_used_tma(self) -> int:
        """1 if the last evaluation staged T by TMA, 0 if by cooperative loads (unaligned T / odd ldT), -1 none."""
        v = ctypes.c_int()
        self._check(_lib.tf_ctx_eval_path(self._h, ctypes.byref(v)))
        return v.value

    def set_cg_grid(self, nblocks: int):
        """Grid size of the persistent CG / matvec kernel (0 = default; > 0: that many blocks, grid kernel)."""
        self._check(_lib.tf_ctx_set_cg_grid(self._h, int(nblocks)))

    def eval_fell_back(self) -> int:
        """1 if the last evaluation ran the guarded Pi form and reran the residual form, 0 if the Pi form held,
        -1 if the last evaluation did not run the Pi form."""
        v = ctypes.c_int()
        self._check(_lib.tf_ctx_eval_fallback(self._h, ctypes.byref(v)))
        return v.value

    def set_timing(self, enable: bool):
        self._check(_lib.tf_ctx_set_timing(self._h, int(bool(enable))))

    def kernel_stats(self, reset: bool = True):
        """(summed fused-eval kernel ms, number of fused-eval launches, total kernel launches)."""
        ms = ctypes.c_double()
        ne = ctypes.c_int64()
        nt = ctypes.c_int64()
        self._check(_lib.tf_ctx_kernel_stats(self._h, ctypes.byref(ms), ctypes.byref(ne), ctypes.byref(nt),
                                             int(bool(reset))))
        return ms.value, ne.value, nt.value


def dims_of(cfg_or_I, J=None, K=None, R=None, **kw) -> Dims:
    if J is None:
        c = cfg_or_I
        return Dims(c.I, c.J, c.K, c.R, **kw)
    return Dims(cfg_or_I, J, K, R, **kw)
