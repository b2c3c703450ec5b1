"""Explicit (dense) objects of the paper for tiny inputs — TEST INFRASTRUCTURE ONLY.

Every function here materialises what the paper defines, with plain loops or
one numpy library primitive per step, so that it can be checked against the
text by eye. Nothing here is used at sizes where a dense object would not fit.

  unfold          Alg. Unfolding, printed example 874-1108
  kron / khatri_rao   Kronecker and Khatri-Rao products
  jacobian_entrywise  J_f from Lemma partialf, rows in storage order
  jacobian_kronecker  J_f from Lemma kronecker, rows in the paper's
                      order (multi-index increasing, last index fastest)
  mttkrp_bruteforce   T_(l) (W^(L) ⊙ ... ⊙ W^(l+1) ⊙ W^(l-1) ⊙ ... ⊙ W^(1)) (Kolda's
                      unfolding formula; gradient thm 2639-2642)
"""
from __future__ import annotations

import numpy as np


def tensor_from_storage(flat, I, J, K) -> np.ndarray:
    """t[i, j, k] array from the first-index-fastest flat storage T[i + I*(j + J*k)]."""
    return np.asarray(flat, dtype=np.float64).reshape(K, J, I).transpose(2, 1, 0).copy()


def storage_from_tensor(t: np.ndarray) -> np.ndarray:
    """Flat first-index-fastest storage of t[i, j, k]."""
    return np.ascontiguousarray(t.transpose(2, 1, 0)).reshape(-1)


def unfold(t: np.ndarray, mode: int) -> np.ndarray:
    """T_(mode) by Alg. Unfolding: mode-`mode` fibers as columns, the remaining indices
    running with the lowest one fastest. mode ∈ {1, 2, 3}."""
    I, J, K = t.shape
    if mode == 1:
        cols = [t[:, j, k] for k in range(K) for j in range(J)]
    elif mode == 2:
        cols = [t[i, :, k] for k in range(K) for i in range(I)]
    elif mode == 3:
        cols = [t[i, j, :] for j in range(J) for i in range(I)]
    else:
        raise ValueError(mode)
    return np.stack(cols, axis=1)


def kron(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Kronecker product [a_11 B, a_12 B, ...], written out."""
    a = np.atleast_2d(a.reshape(a.shape[0], -1))
    b = np.atleast_2d(b.reshape(b.shape[0], -1))
    k, l = a.shape
    m, n = b.shape
    out = np.zeros((k * m, l * n))
    for p in range(k):
        for q in range(l):
            out[p * m:(p + 1) * m, q * n:(q + 1) * n] = a[p, q] * b
    return out


def khatri_rao(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """A ⊙ B = [A_:1 ⊗ B_:1, ..., A_:n ⊗ B_:n]."""
    assert a.shape[1] == b.shape[1]
    return np.concatenate([kron(a[:, r:r + 1], b[:, r:r + 1]) for r in range(a.shape[1])], axis=1)


def mttkrp_bruteforce(t: np.ndarray, A, B, C, mode: int) -> np.ndarray:
    """T_(l) times the reversed Khatri-Rao product of the other factors."""
    if mode == 1:
        return unfold(t, 1) @ khatri_rao(C, B)
    if mode == 2:
        return unfold(t, 2) @ khatri_rao(C, A)
    if mode == 3:
        return unfold(t, 3) @ khatri_rao(B, A)
    raise ValueError(mode)


def factors_from_w(w, I, J, K, R):
    w = np.asarray(w, dtype=np.float64).reshape(-1)
    A = w[:I * R].reshape(R, I).T
    B = w[I * R:(I + J) * R].reshape(R, J).T
    C = w[(I + J) * R:].reshape(R, K).T
    return A, B, C


def jacobian_entrywise(w, I, J, K, R) -> np.ndarray:
    """J_f with rows in storage order (row i + I*(j + J*k)) and columns in w order;
    entry d f_ijk / d w^(l)_{i' r} = -prod_{l != l'} w (Lemma partialf)."""
    A, B, C = factors_from_w(w, I, J, K, R)
    Jm = np.zeros((I * J * K, R * (I + J + K)))
    for k in range(K):
        for j in range(J):
            for i in range(I):
                row = i + I * (j + J * k)
                for r in range(R):
                    Jm[row, r * I + i] = -B[j, r] * C[k, r]
                    Jm[row, I * R + r * J + j] = -A[i, r] * C[k, r]
                    Jm[row, (I + J) * R + r * K + k] = -A[i, r] * B[j, r]
    return Jm


def jacobian_kronecker(w, I, J, K, R) -> np.ndarray:
    """J_f = [df/dW^(1), df/dW^(2), df/dW^(3)] with df/dw_r^(l') = -w_r^(1) ⊗ ... ⊗ I ⊗ ... ⊗ w_r^(L)
    (Lemma kronecker); rows in the paper's order (k fastest)."""
    A, B, C = factors_from_w(w, I, J, K, R)
    blocks = []
    for r in range(R):
        blocks.append(-kron(kron(np.eye(I), B[:, r:r + 1]), C[:, r:r + 1]))
    for r in range(R):
        blocks.append(-kron(kron(A[:, r:r + 1], np.eye(J)), C[:, r:r + 1]))
    for r in range(R):
        blocks.append(-kron(kron(A[:, r:r + 1], B[:, r:r + 1]), np.eye(K)))
    return np.concatenate(blocks, axis=1)


def paper_row_to_storage_row(I, J, K) -> np.ndarray:
    """perm such that J_storage = J_paper[perm]: storage row i + I(j + Jk) <- paper row k + K(j + J i)."""
    perm = np.empty(I * J * K, dtype=np.int64)
    for k in range(K):
        for j in range(J):
            for i in range(I):
                perm[i + I * (j + J * k)] = k + K * (j + J * i)
    return perm


def residual(T_flat, w, I, J, K, R) -> np.ndarray:
    """f(w) in storage order: t_ijk - sum_r a_ir b_jr c_kr, plain loops."""
    A, B, C = factors_from_w(w, I, J, K, R)
    T_flat = np.asarray(T_flat, dtype=np.float64).reshape(-1)
    out = np.empty(I * J * K)
    for k in range(K):
        for j in range(J):
            for i in range(I):
                out[i + I * (j + J * k)] = T_flat[i + I * (j + J * k)] - sum(A[i, r] * B[j, r] * C[k, r]
                                                                            for r in range(R))
    return out
