"""MLSVD compression oracle (NEXT #3 of SURVEY.md §8f) — TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline /
`--impl reference` leg may import this module. It shares no code with the CUDA
path (`paper_2110_05997_b200`) and never imports it.

What it computes, step by step in the paper's order (fp64 numpy; one library
primitive per step — a matmul, `numpy.linalg.eigh` — no blocking or fusion):

  unfolding_gram      T_(l) T_(l)^T from the explicit unfolding (Alg. Unfolding,
                      PAPER.md:857-872), the matrix whose eigenvectors are the
                      left singular vectors of T_(l) (Remark MLSVD-SVD 4446-4448,
                      Lemma svd-transpose 4434-4436, Thm svd-transpose 4442-4444)
  gram_entry          one entry of that Gram by its definition: the inner product
                      of two mode-l hyperslices
  mlsvd               Alg. MLSVD with each SVD taken through
                      the Gram (Remark MLSVD-SVD) and truncated to P_l = min(I_l, R)
                      singular values; singular values sorted
                      decreasingly (Thm MLSVD item 3, 1300); core
                      S = (U1^T, U2^T, U3^T)·T
  core_unfolding      the same core by Thm unfolding-formula (PAPER.md:1282-1285,
                      1312-1313): S_(1) = U1^T T_(1) (U3 ⊗ U2), with an explicit
                      Kronecker product (tiny inputs)
  truncation_ranks    Alg. Compression: the smallest R~_l with
                      sum_{r>R~} sigma_r^2 / sum_{r<=P} sigma_r^2 < mlsvd_tol / L
  compress            Alg. Compression: MLSVD, ranks, truncated U~ and S~
  truncation_error    ||S - S~|| / ||S|| for a truncation shape (Table 4.5, 2970-3021)
  energy_init         the MLSVD-energy initialisation: the R
                      core entries of largest magnitude, S0 = sum_r s_j e ⊗ e ⊗ e
  uncompress          W~_l = U_l W_l
  st_mlsvd            Alg. ST-MLSVD, the sequentially truncated
                      variant Tensor Fox can switch to (1439)

Readings (R23-R26):
  R23 sign of each singular vector: the paper fixes none (any sign gives an SVD);
      we make the entry of largest magnitude of every column of U_l positive
      (first such entry on ties). Only sign-invariant quantities are compared
      across implementations otherwise.
  R24 `rel_error` in Alg. Compression uses R~_l = i (the loop variable); the loop
      always ends because the error at i = P_l is 0 < tol/L.
  R25 the energy initialisation takes the R entries of largest |s| (the
      "brightest" squares of the warming-up example, 3030-3035, whose choice
      s111, s212, s122 is exactly the three largest magnitudes); ties are broken
      by storage order (first index fastest); the coefficient s goes on mode 1.
  R26 the truncated SVD computes the singular values P_l = min(I_l, R) only
      (PAPER.md:1424, 2559), so the relative error in Alg. Compression is
      measured against sum_{r<=P_l} sigma_r^2 (as printed, 2561).
  R32 ST-MLSVD's truncation: the paper gives no rank rule for it; each step
      applies Alg. Compression's rule (tail < mlsvd_tol / L) to that step's
      singular values.

Pins: tests/test_mlsvd_pins.py (Table 4.5 to its 8 printed digits, the printed
core magnitudes 2934-2952, the 0.0153 initial error 3030, the 3.85e-14 truncation
error 2926, Thm MLSVD properties 1296-1301 and 1378-1386, L=2 case = SVD
(1374-1376, numpy SVD), Thm SVD-truncation 1392-1396, Thm energy-mlsvd 1400-1405,
Remark mlsvd-cpd 1346-1352 on exact-rank tensors).
"""
from __future__ import annotations

import numpy as np

from . import jacobian as jac


def _t(T_flat, I, J, K):
    return jac.tensor_from_storage(T_flat, I, J, K)


def unfolding_gram(T_flat, I, J, K, mode: int) -> np.ndarray:
    """T_(mode) T_(mode)^T (I_mode × I_mode) from the explicit unfolding (small/medium inputs)."""
    X = jac.unfold(_t(T_flat, I, J, K), mode)
    return X @ X.T


def gram_entry(T_flat, I, J, K, mode: int, p: int, q: int) -> float:
    """<S_{i_l=p}, S_{i_l=q}>: the (p, q) entry of T_(l) T_(l)^T as the inner product of two
    hyperslices (PAPER.md:1293 defines them; row p of T_(l) is the hyperslice i_l = p), summed in
    extended precision. Works at any size: only the two hyperslices are read."""
    t = np.asarray(T_flat, dtype=np.float64).reshape(K, J, I)   # t[k, j, i]
    if mode == 1:
        a, b = t[:, :, p], t[:, :, q]
    elif mode == 2:
        a, b = t[:, p, :], t[:, q, :]
    else:
        a, b = t[p], t[q]
    return float(np.sum(a.astype(np.longdouble) * b.astype(np.longdouble)))


def _sign_fix(U: np.ndarray) -> np.ndarray:
    """Reading R23: the largest-magnitude entry of each column is made positive."""
    U = U.copy()
    for c in range(U.shape[1]):
        i = int(np.argmax(np.abs(U[:, c])))
        if U[i, c] < 0:
            U[:, c] = -U[:, c]
    return U


def mode_svd(G: np.ndarray, P: int):
    """Left singular vectors and singular values of T_(l) from its Gram G = T_(l) T_(l)^T:
    eigenvectors of G, sigma = sqrt(|lambda|), ordered by |lambda| decreasing (Lemma svd-transpose,
    Thm svd-transpose, Remark MLSVD-SVD), truncated to the first P."""
    lam, V = np.linalg.eigh(G)
    order = np.argsort(-np.abs(lam), kind="stable")
    lam = lam[order][:P]
    V = V[:, order][:, :P]
    return _sign_fix(V), np.sqrt(np.abs(lam)), lam


def multilinear(T_flat, I, J, K, M1, M2, M3) -> np.ndarray:
    """(M1, M2, M3)·T with s_abc = sum_ijk m1_ai m2_bj m3_ck t_ijk (multilinear multiplication,
    PAPER.md:1124-1170 for one mode); returns s[a, b, c]. M_l is (rows × I_l)."""
    t = _t(T_flat, I, J, K)
    return np.einsum("ai,bj,ck,ijk->abc", M1, M2, M3, t, optimize=True)


def core_unfolding(T_flat, I, J, K, U1, U2, U3) -> np.ndarray:
    """S = (U1^T, U2^T, U3^T)·T through Thm unfolding-formula:
    S_(1) = U1^T · T_(1) · (U3 ⊗ U2) (real case: the conjugates are the matrices themselves);
    returned as s[a, b, c] by folding S_(1) back (columns ordered b fastest, then c)."""
    t = _t(T_flat, I, J, K)
    S1 = U1.T @ jac.unfold(t, 1) @ jac.kron(U3, U2)
    P1, P2, P3 = U1.shape[1], U2.shape[1], U3.shape[1]
    s = np.empty((P1, P2, P3))
    for c in range(P3):
        for b in range(P2):
            s[:, b, c] = S1[:, b + P2 * c]
    return s


def mlsvd(T_flat, I, J, K, R: int):
    """Alg. MLSVD with each mode's truncated SVD of P_l = min(I_l, R) singular values.
    Returns dict(U=[U1, U2, U3], sigma=[..], lam=[..], S=s[a,b,c], P=(P1, P2, P3))."""
    dims = (I, J, K)
    Us, sig, lams = [], [], []
    for mode in (1, 2, 3):
        P = min(dims[mode - 1], R)
        U, s, lam = mode_svd(unfolding_gram(T_flat, I, J, K, mode), P)
        Us.append(U)
        sig.append(s)
        lams.append(lam)
    S = multilinear(T_flat, I, J, K, Us[0].T, Us[1].T, Us[2].T)
    return {"U": Us, "sigma": sig, "lam": lams, "S": S, "P": tuple(u.shape[1] for u in Us)}


def truncation_ranks(sigmas, mlsvd_tol: float):
    """Alg. Compression: for each mode the first i = 1..P_l with
    rel_error = sum_{r=i+1}^{P_l} sigma_r^2 / sum_{r=1}^{P_l} sigma_r^2 < mlsvd_tol / L."""
    L = len(sigmas)
    ranks = []
    for s in sigmas:
        s2 = np.asarray(s, dtype=np.float64) ** 2
        total = s2.sum()
        P = len(s2)
        chosen = P
        for i in range(1, P + 1):
            rel_error = s2[i:].sum() / total if total > 0 else 0.0
            if rel_error < mlsvd_tol / L:
                chosen = i
                break
        ranks.append(chosen)
    return tuple(ranks)


def compress(T_flat, I, J, K, R: int, mlsvd_tol: float):
    """Alg. Compression: MLSVD, truncation ranks, U~_l = first R~_l columns, S~ = S[:R~1, :R~2, :R~3]."""
    m = mlsvd(T_flat, I, J, K, R)
    Rt = truncation_ranks(m["sigma"], mlsvd_tol)
    Ut = [m["U"][l][:, :Rt[l]] for l in range(3)]
    St = m["S"][:Rt[0], :Rt[1], :Rt[2]]
    return {"U": Ut, "S": St, "ranks": Rt, "sigma": m["sigma"], "full": m}


def truncation_error(S: np.ndarray, shape) -> float:
    """||S - S~|| / ||S|| with S~ the leading shape[0]×shape[1]×shape[2] block, embedded with zeros
    (PAPER.md:2553 footnote; Table 4.5)."""
    a, b, c = shape
    St = np.zeros_like(S)
    St[:a, :b, :c] = S[:a, :b, :c]
    return float(np.linalg.norm(S - St) / np.linalg.norm(S))


def energy_init(S: np.ndarray, R: int):
    """MLSVD-energy initialisation (reading R25): W1[:, r] = s_j e_{j1},
    W2[:, r] = e_{j2}, W3[:, r] = e_{j3} for the R multi-indexes j of largest |s|.
    Returns (W1, W2, W3, multi-indexes)."""
    P1, P2, P3 = S.shape
    flat = [(abs(S[a, b, c]), a + P1 * (b + P2 * c), (a, b, c))
            for c in range(P3) for b in range(P2) for a in range(P1)]
    flat.sort(key=lambda e: (-e[0], e[1]))
    picks = [e[2] for e in flat[:R]]
    W1, W2, W3 = np.zeros((P1, R)), np.zeros((P2, R)), np.zeros((P3, R))
    for r, (a, b, c) in enumerate(picks):
        W1[a, r] = S[a, b, c]
        W2[b, r] = 1.0
        W3[c, r] = 1.0
    return W1, W2, W3, picks


def uncompress(Us, Ws):
    """W~_l = U_l W_l for each mode."""
    return [U @ W for U, W in zip(Us, Ws)]


def normalize_cpd(Ws):
    """Tensor Fox's output form (flow chart): factors with unit columns and the
    diagonal Lambda, T ≈ sum_r lambda_r w_r^(1) ⊗ w_r^(2) ⊗ w_r^(3), lambda_r = prod_l ||W~_l[:, r]||.
    A zero column keeps lambda_r = 0 and is left as it is."""
    lam = np.ones(Ws[0].shape[1])
    out = []
    for W in Ws:
        nrm = np.sqrt(np.sum(W * W, axis=0))
        lam = lam * nrm
        out.append(np.where(nrm > 0, W / np.where(nrm > 0, nrm, 1.0), W))
    return out, lam


def st_mlsvd(T_flat, I, J, K, R: int, mlsvd_tol: float):
    """Alg. ST-MLSVD: S^(0) = T; for l = 1, 2, 3 the SVD of the current unfolding
    S^(l-1)_(l) (through its Gram, truncated to P_l = min(I_l, R) singular values), the rank R~_l by the rule of
    Alg. Compression applied to that step's singular values (reading R32), and S^(l) = the mode-l product of
    S^(l-1) with U~_l^T (i.e. S^(l)_(l) = Sigma~ V~^T). Returns dict(U=[U~_l], Ufull=[U_l (P_l cols)],
    sigma=[sigma_l], ranks, S=S^(3))."""
    S = _t(T_flat, I, J, K)
    Us, Ufull, sig, ranks = [], [], [], []
    for mode in (1, 2, 3):
        n = S.shape[mode - 1]
        P = min(n, R)
        X = jac.unfold(S, mode)
        U, s, _ = mode_svd(X @ X.T, P)
        r = truncation_ranks([s], mlsvd_tol / 3)[0]   # the per-mode rule: tail < mlsvd_tol / L, L = 3
        Ut = U[:, :r]
        if mode == 1:
            S = np.einsum("ia,ijk->ajk", Ut, S)
        elif mode == 2:
            S = np.einsum("jb,ajk->abk", Ut, S)
        else:
            S = np.einsum("kc,abk->abc", Ut, S)
        Us.append(Ut)
        Ufull.append(U)
        sig.append(s)
        ranks.append(r)
    return {"U": Us, "Ufull": Ufull, "sigma": sig, "ranks": tuple(ranks), "S": S}
