"""CP-ALS oracle (NEXT #4 of SURVEY.md §8f) — TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline /
`--impl reference` leg may import this module. It shares no code with the CUDA
path (`paper_2110_05997_b200`) and never imports it.

Alg. ALS for L = 3, each factor update written as the paper
derives it:

    W^(l) <- T_(l) (⊙_{l' != l} W^(l'))  ((*_{l' != l} W^(l')^T W^(l'))^dagger)

with the reversed Khatri–Rao order of Thm unfolding-formula2 (T_(1) (C ⊙ B),
T_(2) (C ⊙ A), T_(3) (B ⊙ A)), the pseudo-inverse of the
Khatri–Rao product from Thm special-products items 11-12,
and the modes updated in order 1, 2, 3 within a sweep, each with the newest
factors. Explicit unfoldings and Khatri–Rao products (oracle/jacobian.py), one
numpy primitive per step (matmul, `numpy.linalg.pinv`), fp64.

Reading R30: the paper does not fix the pseudo-inverse cut-off; we
take numpy's pinv rule — eigen/singular values below 1e-15 × the largest are
treated as zero — on the symmetric R × R matrix V.

Pins: tests/test_als_pins.py (the least-squares optimality of each update —
the mode-l block of grad F from oracle.cpd_eval vanishes after updating mode l;
equality with numpy.linalg.lstsq on the materialised Khatri–Rao system; the
fixed point at the true factors of an exact-rank tensor; monotone F per update).
"""
from __future__ import annotations

import numpy as np

from . import jacobian as jac


def _factors(w, I, J, K, R):
    w = np.asarray(w, dtype=np.float64).reshape(-1)
    return [w[:I * R].reshape(R, I).T.copy(), w[I * R:(I + J) * R].reshape(R, J).T.copy(),
            w[(I + J) * R:].reshape(R, K).T.copy()]


def _pack(Ws):
    return np.concatenate([W.T.reshape(-1) for W in Ws])


def pinv_sym(V: np.ndarray) -> np.ndarray:
    """Pseudo-inverse of the symmetric R × R matrix V (numpy.linalg.pinv, rcond 1e-15; reading R30)."""
    return np.linalg.pinv(V, rcond=1e-15, hermitian=True)


def als_update(T_flat, Ws, mode: int, I, J, K):
    """One factor update of Alg. ALS: W^(mode) = T_(mode) KR (V^dagger)."""
    t = jac.tensor_from_storage(T_flat, I, J, K)
    A, B, C = Ws
    if mode == 1:
        KR, V = jac.khatri_rao(C, B), (C.T @ C) * (B.T @ B)
    elif mode == 2:
        KR, V = jac.khatri_rao(C, A), (C.T @ C) * (A.T @ A)
    else:
        KR, V = jac.khatri_rao(B, A), (B.T @ B) * (A.T @ A)
    M = jac.unfold(t, mode) @ KR
    out = list(Ws)
    out[mode - 1] = M @ pinv_sym(V)
    return out


def als(T_flat, w0, I, J, K, R, sweeps: int):
    """`sweeps` sweeps of Alg. ALS from w0; returns (w, F after every update [3*sweeps])."""
    Ws = _factors(w0, I, J, K, R)
    t = jac.tensor_from_storage(T_flat, I, J, K)
    fs = []
    for _ in range(sweeps):
        for mode in (1, 2, 3):
            Ws = als_update(T_flat, Ws, mode, I, J, K)
            rec = np.einsum("ir,jr,kr->ijk", *Ws)
            fs.append(0.5 * float(np.sum((t - rec) ** 2)))
    return _pack(Ws), np.array(fs)


def mttkrp(T_flat, Ws, mode: int, I, J, K):
    """T_(mode) times the reversed Khatri–Rao product of the other factors (Thm unfolding-formula2)."""
    return jac.mttkrp_bruteforce(jac.tensor_from_storage(T_flat, I, J, K), *Ws, mode)
