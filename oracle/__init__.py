"""CPU oracle for the Tensor Fox dGN evaluation hot path (arxiv 2110.05997).

TEST INFRASTRUCTURE ONLY. Only `tests/`, `__graft_entry__.smoke()` and
`bench.py`'s cpu_baseline / `--impl reference` leg may import this package.
It shares no code with `paper_2110_05997_b200` (the CUDA path) and never
imports it; the CUDA path never imports this.

Contents
  * `oracle.c` (compiled here with gcc into `liboracle.so`): the definitions of
    F, grad F = J_f^T f, the plain J-then-J^T Gauss-Newton matvec, Grams, the
    Hadamard chains, Thm Hv, diag(J^T J) and Alg. CG-dGN, all accumulated in
    80-bit long double (see the C header for citations).
  * `jacobian.py`: the explicit Jacobian on tiny inputs, built twice from two
    different statements of the paper (Lemma partialf, entrywise; Lemma
    kronecker, Kronecker-product columns), plus explicit unfoldings and
    Khatri-Rao products (Alg. Unfolding; Kolda's unfolding formula).
  * `mlsvd.py`: the MLSVD compression stage (NEXT #3): unfolding Grams, the
    truncated MLSVD through them, Alg. Compression, the MLSVD-energy
    initialisation and uncompression (numpy fp64, eigh as the SVD primitive).

Pins (tests/test_oracle_pins.py, `-m "not gpu"`) tie every function to the
paper or to mathematics; the list, and any function left "parity unpinned",
is kept in DESIGN.md §3.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

_d = ctypes.POINTER(ctypes.c_double)
_i64 = ctypes.c_int64


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so (gcc -O2, no -ffast-math, OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            L = ctypes.CDLL(build())
            L.oracle_eval.argtypes = [_i64] * 4 + [_d] * 4 + [_d] * 4 + [ctypes.c_int]
            L.oracle_slice_eval.argtypes = [_i64, _i64, _i64, _d, _i64, _i64, _d, _d, _i64, _d, _i64, _d, _d]
            L.oracle_gn_matvec_plain.argtypes = [_i64] * 4 + [_d] * 4 + [ctypes.c_double, _d, _d, ctypes.c_int]
            L.oracle_grams.argtypes = [_i64] * 4 + [_d] * 4
            L.oracle_pi.argtypes = [_i64, _d, _d]
            L.oracle_gn_matvec_hv.argtypes = [_i64] * 4 + [_d] * 4 + [ctypes.c_double, _d, _d]
            L.oracle_reg_gamma.argtypes = [_i64] * 4 + [_d] * 4
            L.oracle_jtj_diag.argtypes = [_i64] * 4 + [_d] * 4
            L.oracle_cg.argtypes = ([_i64] * 4 + [_d] * 4 + [ctypes.c_double, _d, ctypes.c_int, ctypes.c_double,
                                    ctypes.c_int] + [_d] * 5 + [ctypes.POINTER(ctypes.c_int)])
            L.oracle_dgn_stop.argtypes = [ctypes.c_int, _d, ctypes.c_int] + [ctypes.c_double] * 4
            L.oracle_dgn_stop.restype = ctypes.c_int
            L.oracle_dgn.argtypes = ([_i64] * 4 + [_d, _d, ctypes.c_int, ctypes.c_double, ctypes.c_double] +
                                     [ctypes.c_int] * 3 + [ctypes.POINTER(ctypes.c_int)] * 3 + [_d, _d, ctypes.c_int])
            _lib = L
    return _lib


def _p(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(_d)


def _np(x) -> np.ndarray:
    """torch tensor or array -> contiguous float64 numpy array (host)."""
    if hasattr(x, "detach"):
        x = x.detach().cpu().numpy()
    return np.ascontiguousarray(np.asarray(x, dtype=np.float64))


def _split(w, I, J, K, R):
    w = _np(w).reshape(-1)
    assert w.size == R * (I + J + K), (w.size, R, I, J, K)
    return w[:R * I].copy(), w[R * I:R * (I + J)].copy(), w[R * (I + J):].copy()


def cpd_eval(T, w, I, J, K, R, nthreads: int = 0):
    """(F, grad) at w for the I×J×K tensor T (any array whose flat order is T[i + I*(j + J*k)]).

    Returns f (float) and grad (n,) in w-layout [vec dF/dA; vec dF/dB; vec dF/dC].
    """
    T = _np(T).reshape(-1)
    assert T.size == I * J * K
    A, B, C = _split(w, I, J, K, R)
    f = ctypes.c_double()
    gA, gB, gC = np.zeros(I * R), np.zeros(J * R), np.zeros(K * R)
    rc = lib().oracle_eval(I, J, K, R, _p(T), _p(A), _p(B), _p(C), ctypes.byref(f), _p(gA), _p(gB), _p(gC),
                           nthreads)
    if rc:
        raise RuntimeError(f"oracle_eval rc={rc}")
    return f.value, np.concatenate([gA, gB, gC])


def slice_eval(S, x, X, Y):
    """One slice of T with its fixed-index factor row x (R,), the other factors X (n1,R), Y (n2,R)
    (numpy, any layout). S is (n1, n2). Returns (share of F, gradient row of the fixed index)."""
    S = np.asarray(S, dtype=np.float64)
    X = np.asfortranarray(np.asarray(X, dtype=np.float64))
    Y = np.asfortranarray(np.asarray(Y, dtype=np.float64))
    x = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    n1, n2 = S.shape
    R = x.size
    s1, s2 = S.strides[0] // 8, S.strides[1] // 8
    base = S
    f = ctypes.c_double()
    g = np.zeros(R)
    rc = lib().oracle_slice_eval(n1, n2, R, base.ctypes.data_as(_d), s1, s2, _p(x),
                                 X.ctypes.data_as(_d), X.shape[0], Y.ctypes.data_as(_d), Y.shape[0],
                                 ctypes.byref(f), _p(g))
    if rc:
        raise RuntimeError(f"oracle_slice_eval rc={rc}")
    return f.value, g


def _damp(damp):
    return None if damp is None else _np(damp).reshape(-1)


def gn_matvec_plain(w, v, lam, I, J, K, R, nthreads: int = 0, damp=None):
    """(J^T J + lam D) v via u = J v then J^T u (Lemma partialf), O(IJKR). D = diag(damp) per (mode, r)."""
    A, B, C = _split(w, I, J, K, R)
    v = _np(v).reshape(-1)
    y = np.zeros_like(v)
    d = _damp(damp)
    rc = lib().oracle_gn_matvec_plain(I, J, K, R, _p(A), _p(B), _p(C), _p(v), float(lam),
                                      None if d is None else _p(d), _p(y), nthreads)
    if rc:
        raise RuntimeError(f"oracle_gn_matvec_plain rc={rc}")
    return y


def grams(w, I, J, K, R):
    """[A^T A | B^T B | C^T C], each R×R column-major, flattened (3R²,)."""
    A, B, C = _split(w, I, J, K, R)
    g = np.zeros(3 * R * R)
    lib().oracle_grams(I, J, K, R, _p(A), _p(B), _p(C), _p(g))
    return g


def hadamard_chains(grams_, R):
    """[Pi1 | Pi2 | Pi3 | Pi12 | Pi13 | Pi23] (6R²,) from [piA | piB | piC]."""
    g = _np(grams_).reshape(-1)
    out = np.zeros(6 * R * R)
    lib().oracle_pi(R, _p(g), _p(out))
    return out


def gn_matvec_hv(w, v, lam, I, J, K, R, damp=None):
    """(J^T J + lam D) v by Thm Hv; D = diag(damp) per (mode, r), None = I."""
    A, B, C = _split(w, I, J, K, R)
    v = _np(v).reshape(-1)
    y = np.zeros_like(v)
    d = _damp(damp)
    lib().oracle_gn_matvec_hv(I, J, K, R, _p(A), _p(B), _p(C), _p(v), float(lam), None if d is None else _p(d),
                              _p(y))
    return y


def reg_gamma(w, I, J, K, R):
    """Tensor Fox's diagonal regularizer gamma = [gamma_X | gamma_Y | gamma_Z], 3R."""
    A, B, C = _split(w, I, J, K, R)
    g = np.zeros(3 * R)
    lib().oracle_reg_gamma(I, J, K, R, _p(A), _p(B), _p(C), _p(g))
    return g


def jtj_diag(w, I, J, K, R):
    A, B, C = _split(w, I, J, K, R)
    d = np.zeros(R * (I + J + K))
    lib().oracle_jtj_diag(I, J, K, R, _p(A), _p(B), _p(C), _p(d))
    return d


def cg(w, rhs, lam, maxiter, I, J, K, R, tol=0.0, jacobi=False, history=False, damp=None):
    """Alg. CG-dGN on (J^T J + lam D); D = diag(damp) per (mode, r), None = I.
    Returns dict(x, iters, r2, alpha, beta[, x_hist])."""
    A, B, C = _split(w, I, J, K, R)
    rhs = _np(rhs).reshape(-1)
    n = rhs.size
    x = np.zeros(n)
    m = max(int(maxiter), 1)
    xh = np.zeros(m * n) if history else None
    r2, al, be = np.zeros(m), np.zeros(m), np.zeros(m)
    it = ctypes.c_int()
    d = _damp(damp)
    rc = lib().oracle_cg(I, J, K, R, _p(A), _p(B), _p(C), _p(rhs), float(lam), None if d is None else _p(d),
                         int(maxiter), float(tol),
                         int(bool(jacobi)), _p(x), _p(xh) if history else None, _p(r2), _p(al), _p(be),
                         ctypes.byref(it))
    out = {"x": x, "iters": it.value, "r2": r2[:it.value], "alpha": al[:it.value], "beta": be[:it.value],
           "status": rc}
    if history:
        out["x_hist"] = xh.reshape(m, n)[:it.value]
    return out


def dgn(T, w0, I, J, K, R, cg_iters, maxiter=None, tol=1e-6, mu0=0.0, use_gamma=True, jacobi=True, balance=True,
        nthreads: int = 0):
    """The dGN outer loop of Tensor Fox from w0 with the given per-iteration CG budgets.
    Returns dict(w, iters, reason, f, hist[iters, 5] = [F, rel_err, mu, g, ||x||])."""
    T = _np(T).reshape(-1)
    w = _np(w0).reshape(-1).copy()
    cgi = np.ascontiguousarray(np.asarray(cg_iters, dtype=np.int32))
    m = int(maxiter if maxiter is not None else cgi.size)
    assert cgi.size >= m
    hist = np.zeros(5 * max(m, 1))
    it, why = ctypes.c_int(), ctypes.c_int()
    f = ctypes.c_double()
    lib().oracle_dgn(I, J, K, R, _p(T), _p(w), m, float(tol), float(mu0), int(use_gamma), int(jacobi), int(balance),
                     cgi.ctypes.data_as(ctypes.POINTER(ctypes.c_int)), ctypes.byref(it), ctypes.byref(why),
                     ctypes.byref(f), _p(hist), nthreads)
    return {"w": w, "iters": it.value, "reason": why.value, "f": f.value, "hist": hist.reshape(-1, 5)[:it.value]}


def dgn_stop(k, rel, maxiter, tol, step, ginf, normT2):
    """The dGN stopping rule at iteration k: the first condition 1..7 that holds, or 0.
    rel = relative errors after 0..k iterations (at least k + 1 values)."""
    r = np.ascontiguousarray(np.asarray(rel, dtype=np.float64))
    assert r.size >= k + 1 and k >= 1
    return int(lib().oracle_dgn_stop(int(k), _p(r), int(maxiter), float(tol), float(step), float(ginf), float(normT2)))
