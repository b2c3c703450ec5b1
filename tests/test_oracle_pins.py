"""Pins of the CPU oracle to what the paper and mathematics fix (runs without a GPU).

Each test ties one oracle function to something other than itself: values the
paper prints (tests/golden/, cited), closed forms, exact identities, a second
derivation from another statement of the paper, or brute force on tiny inputs.
A plausible slip (dropped term, wrong sign, wrong index or transposed operand)
in the oracle fails at least one of them. DESIGN.md §3 maps pins to functions.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
from oracle import jacobian as jac

U = 2.0 ** -53
RNG = np.random.default_rng(20211012)


def rand_w(I, J, K, R, scale=1.0, rng=RNG):
    return scale * rng.standard_normal(R * (I + J + K))


def dense_T(t):
    return jac.storage_from_tensor(t)


def build_T(A, B, C):
    """t_ijk = sum_r a_ir b_jr c_kr, via einsum (independent of the oracle)."""
    return np.einsum("ir,jr,kr->ijk", A, B, C)


def w_of(A, B, C):
    return np.concatenate([A.T.reshape(-1), B.T.reshape(-1), C.T.reshape(-1)])


def pi_numpy(A, B, C):
    gA, gB, gC = A.T @ A, B.T @ B, C.T @ C
    return gB * gC, gA * gC, gA * gB


# --------------------------------------------------------------------------- layout
def test_storage_and_unfoldings_match_paper_example(golden_dir):
    g = json.load(open(os.path.join(golden_dir, "unfold_3x4x2.json")))
    fs = np.array(g["frontal_slices"], dtype=np.float64)      # [k][i][j]
    t = fs.transpose(1, 2, 0)                                   # t[i, j, k]
    # first-index-fastest storage of this tensor is 1..24
    assert np.array_equal(jac.storage_from_tensor(t), np.arange(1, 25, dtype=np.float64))
    assert np.array_equal(jac.tensor_from_storage(np.arange(1, 25), 3, 4, 2), t)
    assert np.array_equal(jac.unfold(t, 1), np.array(g["T1"]))
    assert np.array_equal(jac.unfold(t, 2), np.array(g["T2"]))
    assert np.array_equal(jac.unfold(t, 3), np.array(g["T3"]))
    # mode-1 product example
    assert np.array_equal(np.array(g["M"]) @ jac.unfold(t, 1), np.array(g["M_T1"]))


def test_khatri_rao_matches_unfolding_formula():
    """Kolda: T = [[A,B,C]] => T_(1) = A (C ⊙ B)^T, T_(2) = B (C ⊙ A)^T, T_(3) = C (B ⊙ A)^T."""
    I, J, K, R = 4, 3, 5, 2
    A, B, C = (RNG.standard_normal((n, R)) for n in (I, J, K))
    t = build_T(A, B, C)
    np.testing.assert_allclose(jac.unfold(t, 1), A @ jac.khatri_rao(C, B).T, rtol=0, atol=1e-13)
    np.testing.assert_allclose(jac.unfold(t, 2), B @ jac.khatri_rao(C, A).T, rtol=0, atol=1e-13)
    np.testing.assert_allclose(jac.unfold(t, 3), C @ jac.khatri_rao(B, A).T, rtol=0, atol=1e-13)


# --------------------------------------------------------------------------- F and grad
@pytest.mark.parametrize("dims", [(5, 4, 3, 3), (2, 7, 3, 2), (6, 1, 4, 5), (3, 3, 3, 1)])
def test_gradient_equals_bruteforce_mttkrp(dims):
    """grad F = W Π − T_(l)(⊙W) with explicit unfolding × materialised Khatri-Rao."""
    I, J, K, R = dims
    t = RNG.standard_normal((I, J, K))
    w = rand_w(I, J, K, R)
    A, B, C = jac.factors_from_w(w, I, J, K, R)
    f, g = oracle.cpd_eval(dense_T(t), w, I, J, K, R)
    P1, P2, P3 = pi_numpy(A, B, C)
    gA = A @ P1 - jac.mttkrp_bruteforce(t, A, B, C, 1)
    gB = B @ P2 - jac.mttkrp_bruteforce(t, A, B, C, 2)
    gC = C @ P3 - jac.mttkrp_bruteforce(t, A, B, C, 3)
    ref = np.concatenate([gA.T.reshape(-1), gB.T.reshape(-1), gC.T.reshape(-1)])
    np.testing.assert_allclose(g, ref, rtol=1e-11, atol=1e-11 * np.abs(ref).max())
    # F by its definition with numpy
    np.testing.assert_allclose(f, 0.5 * np.sum((t - build_T(A, B, C)) ** 2), rtol=1e-12)


def test_gradient_is_JT_times_residual():
    """Lemma gradF: ∇F = J_f^T f, J from Lemma partialf, f by plain loops."""
    I, J, K, R = 4, 3, 2, 3
    T = RNG.standard_normal(I * J * K)
    w = rand_w(I, J, K, R)
    Jm = jac.jacobian_entrywise(w, I, J, K, R)
    r = jac.residual(T, w, I, J, K, R)
    f, g = oracle.cpd_eval(T, w, I, J, K, R)
    np.testing.assert_allclose(g, Jm.T @ r, rtol=1e-12, atol=1e-13)
    np.testing.assert_allclose(f, 0.5 * r @ r, rtol=1e-13)


def test_gradient_central_differences_exact():
    """F is quadratic along every coordinate line (t̃ is linear in each single parameter, Lemma partialf),
    so (F(w+h e_j) − F(w−h e_j)) / 2h = ∂_j F exactly, for any h; use h = 1."""
    I, J, K, R = 5, 4, 3, 2
    T = RNG.standard_normal(I * J * K)
    w = rand_w(I, J, K, R)
    f0, g = oracle.cpd_eval(T, w, I, J, K, R)
    for idx in list(range(0, w.size, 3)) + [w.size - 1]:
        e = np.zeros_like(w)
        e[idx] = 1.0
        fp, _ = oracle.cpd_eval(T, w + e, I, J, K, R)
        fm, _ = oracle.cpd_eval(T, w - e, I, J, K, R)
        fd = (fp - fm) / 2.0
        assert abs(fd - g[idx]) <= 1e-12 * max(abs(fp), abs(fm), 1.0), (idx, fd, g[idx])


def test_zero_residual_and_gradient_at_true_factors_warmup(golden_dir):
    """Warming-up tensor t_ijk = φ(x_i,y_j,z_k) built from φ itself, factors from its closed-form
    rank-3 splitting: F ≈ 0 and ∇F ≈ 0 at the true factors."""
    g = json.load(open(os.path.join(golden_dir, "warmup.json")))
    x = np.array(g["x"])
    y = np.array(g["y"])
    z = np.array(g["z_num"], dtype=np.float64) / g["z_den"]
    X, Y, Z = np.meshgrid(x, y, z, indexing="ij")
    t = (np.cos(1 - X) * np.sin(1 + Y ** 2) - np.sin(1 + X ** 2) * np.exp(X ** 2 + Y ** 2 + Z ** 2)
         - np.cos(X) * np.log(1 + Z))
    A = np.stack([np.cos(1 - x), -np.sin(1 + x ** 2) * np.exp(x ** 2), -np.cos(x)], axis=1)
    B = np.stack([np.sin(1 + y ** 2), np.exp(y ** 2), np.ones_like(y)], axis=1)
    C = np.stack([np.ones_like(z), np.exp(z ** 2), np.log(1 + z)], axis=1)
    I, J, K, R = 6, 5, 4, 3
    w = w_of(A, B, C)
    nT2 = float(np.sum(t * t))
    assert abs(math.sqrt(nT2) - g["norm_T_survey_check"]) < 1e-4
    f, grad = oracle.cpd_eval(dense_T(t), w, I, J, K, R)
    assert f <= (16 * U) ** 2 * nT2, f
    P1, P2, P3 = pi_numpy(A, B, C)
    floor = U * (np.linalg.norm(A @ P1) + np.linalg.norm(B @ P2) + np.linalg.norm(C @ P3))
    assert np.linalg.norm(grad) <= 64 * floor, (np.linalg.norm(grad), floor)
    # and away from the true point the gradient is not small (the test can fail)
    _, g2 = oracle.cpd_eval(dense_T(t), w + 1e-3 * rand_w(I, J, K, R), I, J, K, R)
    assert np.linalg.norm(g2) > 1e6 * floor
    # the paper's printed final CPD fits T to ~5.6e-7 relative error
    Xp, Yp, Zp = (np.array(g[k]) for k in ("printed_X", "printed_Y", "printed_Z"))
    fp, _ = oracle.cpd_eval(dense_T(t), w_of(Xp, Yp, Zp), I, J, K, R)
    rel = math.sqrt(2 * fp / nT2)
    assert 1e-7 < rel < 1e-6, rel


def test_zero_at_true_factors_bottleneck(golden_dir):
    """Bottleneck example: exact rank 3 with R > dims, F = 0, ∇F = 0 at its factors."""
    g = json.load(open(os.path.join(golden_dir, "bottleneck_2x2x2.json")))
    A, B, C = (np.array(g[k]) for k in "ABC")
    t = build_T(A, B, C)
    w = w_of(A, B, C)
    f, grad = oracle.cpd_eval(dense_T(t), w, 2, 2, 2, 3)
    assert f <= 1e-28
    assert np.abs(grad).max() <= 1e-12


@pytest.mark.parametrize("n", [10.0, 100.0, 1000.0])
def test_border_rank_closed_form(n):
    """de Silva–Lim: T = x⊗x⊗y + x⊗y⊗x + y⊗x⊗x, rank-2 T^(n) = n(x+y/n)^{⊗3} − n x^{⊗3}.
    With orthonormal x, y: ‖T − T^(n)‖² = 3/n² + 1/n⁴, so F = ½(3/n² + 1/n⁴)."""
    I, J, K = 3, 4, 2
    e = lambda m, k: np.eye(m)[:, k]
    t = (np.einsum("i,j,k->ijk", e(I, 0), e(J, 0), e(K, 1)) + np.einsum("i,j,k->ijk", e(I, 0), e(J, 1), e(K, 0))
         + np.einsum("i,j,k->ijk", e(I, 1), e(J, 0), e(K, 0)))
    A = np.stack([n * (e(I, 0) + e(I, 1) / n), -n * e(I, 0)], axis=1)
    B = np.stack([e(J, 0) + e(J, 1) / n, e(J, 0)], axis=1)
    C = np.stack([e(K, 0) + e(K, 1) / n, e(K, 0)], axis=1)
    f, _ = oracle.cpd_eval(dense_T(t), w_of(A, B, C), I, J, K, 2)
    ref = 0.5 * (3.0 / n ** 2 + 1.0 / n ** 4)
    assert abs(f - ref) <= 1e-12 * ref, (f, ref)


def test_matmul_tensor_mttkrp_closed_form():
    """Matrix-multiplication tensor M_N: with vec = column stacking,
    t[(i,j),(j,k),(i,k)] = 1, the mode-1 MTTKRP column r is vec(Z_r Y_r^T), Y_r = mat(B_:r), Z_r = mat(C_:r)."""
    N, R = 3, 4
    n = N * N
    t = np.zeros((n, n, n))
    for i in range(N):
        for j in range(N):
            for k in range(N):
                t[i + N * j, j + N * k, i + N * k] = 1.0
    w = rand_w(n, n, n, R)
    A, B, C = jac.factors_from_w(w, n, n, n, R)
    _, g = oracle.cpd_eval(dense_T(t), w, n, n, n, R)
    gA = g[:n * R].reshape(R, n).T
    P1, _, _ = pi_numpy(A, B, C)
    mttkrp = A @ P1 - gA                        # Kolda: ∂F/∂A = A Π^(1) − T_(1)(C ⊙ B)
    for r in range(R):
        Yr = B[:, r].reshape(N, N, order="F")
        Zr = C[:, r].reshape(N, N, order="F")
        np.testing.assert_allclose(mttkrp[:, r], (Zr @ Yr.T).reshape(-1, order="F"), rtol=0, atol=1e-12)


def test_slice_eval_rows_match_full_eval():
    """Sampled-row oracle (one slice per fixed index) agrees with the full evaluation."""
    I, J, K, R = 6, 5, 4, 3
    t = RNG.standard_normal((I, J, K))
    w = rand_w(I, J, K, R)
    A, B, C = jac.factors_from_w(w, I, J, K, R)
    f, g = oracle.cpd_eval(dense_T(t), w, I, J, K, R)
    gA = g[:I * R].reshape(R, I).T
    gB = g[I * R:(I + J) * R].reshape(R, J).T
    gC = g[(I + J) * R:].reshape(R, K).T
    fk = 0.0
    for k in range(K):
        fs, row = oracle.slice_eval(t[:, :, k], C[k], A, B)
        np.testing.assert_allclose(row, gC[k], rtol=1e-13, atol=1e-14)
        fk += fs
    np.testing.assert_allclose(fk, f, rtol=1e-13)
    for i in range(I):
        _, row = oracle.slice_eval(t[i, :, :], A[i], B, C)
        np.testing.assert_allclose(row, gA[i], rtol=1e-13, atol=1e-14)
    for j in range(J):
        _, row = oracle.slice_eval(t[:, j, :], B[j], A, C)
        np.testing.assert_allclose(row, gB[j], rtol=1e-13, atol=1e-14)


def test_eval_sums_over_k_shards():
    """F, gA, gB are sums over frontal-slice shards; gC rows are local."""
    I, J, K, R = 4, 5, 7, 3
    t = RNG.standard_normal((I, J, K))
    w = rand_w(I, J, K, R)
    A, B, C = jac.factors_from_w(w, I, J, K, R)
    f, g = oracle.cpd_eval(dense_T(t), w, I, J, K, R)
    acc_f, acc_AB = 0.0, np.zeros((I + J) * R)
    gC = np.zeros(K * R)
    for k0, k1 in [(0, 3), (3, 4), (4, 7)]:
        ws = w_of(A, B, C[k0:k1])
        fs, gs = oracle.cpd_eval(dense_T(t[:, :, k0:k1]), ws, I, J, k1 - k0, R)
        acc_f += fs
        acc_AB += gs[:(I + J) * R]
        gC.reshape(R, K)[:, k0:k1] = gs[(I + J) * R:].reshape(R, k1 - k0)
    np.testing.assert_allclose(acc_f, f, rtol=1e-13)
    np.testing.assert_allclose(acc_AB, g[:(I + J) * R], rtol=1e-12, atol=1e-13)
    np.testing.assert_allclose(gC, g[(I + J) * R:], rtol=1e-13, atol=1e-14)


# --------------------------------------------------------------------------- Jacobian, Grams, matvec
def test_jacobian_lemma_partialf_equals_lemma_kronecker():
    I, J, K, R = 4, 3, 2, 2
    w = rand_w(I, J, K, R)
    Je = jac.jacobian_entrywise(w, I, J, K, R)
    Jk = jac.jacobian_kronecker(w, I, J, K, R)
    perm = jac.paper_row_to_storage_row(I, J, K)
    np.testing.assert_array_equal(Je, Jk[perm])


def test_grams_and_hadamard_chains():
    """π^(l) = W^T W; Π^(1) = (C⊙B)^T(C⊙B) = π_C ∗ π_B (Thm special-products 11)."""
    I, J, K, R = 5, 4, 3, 3
    w = rand_w(I, J, K, R)
    A, B, C = jac.factors_from_w(w, I, J, K, R)
    g = oracle.grams(w, I, J, K, R)
    np.testing.assert_allclose(g[:R * R].reshape(R, R), A.T @ A, rtol=1e-13)
    np.testing.assert_allclose(g[R * R:2 * R * R].reshape(R, R), B.T @ B, rtol=1e-13)
    np.testing.assert_allclose(g[2 * R * R:].reshape(R, R), C.T @ C, rtol=1e-13)
    p = oracle.hadamard_chains(g, R).reshape(6, R, R)
    KR1, KR2, KR3 = jac.khatri_rao(C, B), jac.khatri_rao(C, A), jac.khatri_rao(B, A)
    np.testing.assert_allclose(p[0], KR1.T @ KR1, rtol=1e-12)
    np.testing.assert_allclose(p[1], KR2.T @ KR2, rtol=1e-12)
    np.testing.assert_allclose(p[2], KR3.T @ KR3, rtol=1e-12)
    np.testing.assert_allclose(p[3], C.T @ C, rtol=1e-13)    # Π^(1,2): product over l ∉ {1,2}
    np.testing.assert_allclose(p[4], B.T @ B, rtol=1e-13)    # Π^(1,3)
    np.testing.assert_allclose(p[5], A.T @ A, rtol=1e-13)    # Π^(2,3)


@pytest.mark.parametrize("lam", [0.0, 1e-3, 2.5])
def test_gn_matvec_against_explicit_jacobian(lam):
    """(J^T J + λI) v: Thm Hv and the plain J-then-J^T route both equal the explicit product (Thm JfT_Jf)."""
    for (I, J, K, R) in [(4, 3, 2, 3), (2, 5, 3, 2), (3, 3, 3, 1)]:
        w = rand_w(I, J, K, R)
        v = RNG.standard_normal(R * (I + J + K))
        Jm = jac.jacobian_entrywise(w, I, J, K, R)
        ref = Jm.T @ (Jm @ v) + lam * v
        sc = np.abs(ref).max()
        np.testing.assert_allclose(oracle.gn_matvec_hv(w, v, lam, I, J, K, R), ref, rtol=1e-12, atol=1e-13 * sc)
        np.testing.assert_allclose(oracle.gn_matvec_plain(w, v, lam, I, J, K, R), ref, rtol=1e-12,
                                   atol=1e-13 * sc)


def test_gn_matvec_plain_vs_hv_medium():
    """The two independent routes agree at a size where the explicit J is not formed."""
    I, J, K, R = 20, 17, 9, 5
    w = rand_w(I, J, K, R)
    v = RNG.standard_normal(R * (I + J + K))
    a = oracle.gn_matvec_hv(w, v, 1e-3, I, J, K, R)
    b = oracle.gn_matvec_plain(w, v, 1e-3, I, J, K, R)
    np.testing.assert_allclose(a, b, rtol=1e-12, atol=1e-13 * np.abs(b).max())


def test_gn_matvec_scaling_null_vectors():
    """JᵀJ is singular: scaling column r of A up and of B down leaves [[A,B,C]]
    unchanged to first order, so J v = 0 and (JᵀJ + λI) v = λ v."""
    I, J, K, R = 6, 5, 4, 3
    lam = 0.37
    w = rand_w(I, J, K, R)
    A, B, C = jac.factors_from_w(w, I, J, K, R)
    for r in range(R):
        VA, VB, VC = np.zeros_like(A), np.zeros_like(B), np.zeros_like(C)
        VA[:, r] = A[:, r]
        VB[:, r] = -B[:, r]
        v = w_of(VA, VB, VC)
        np.testing.assert_allclose(oracle.gn_matvec_plain(w, v, lam, I, J, K, R), lam * v, rtol=0, atol=1e-15)
        y = oracle.gn_matvec_hv(w, v, lam, I, J, K, R)
        scale = np.abs(oracle.gn_matvec_hv(w, np.abs(v), 0.0, I, J, K, R)).max()
        np.testing.assert_allclose(y, lam * v, rtol=0, atol=1e-13 * scale)


def test_gn_matvec_symmetric_psd_and_diagonal():
    I, J, K, R = 7, 6, 5, 4
    w = rand_w(I, J, K, R)
    n = R * (I + J + K)
    u, v = RNG.standard_normal(n), RNG.standard_normal(n)
    Hu = oracle.gn_matvec_hv(w, u, 0.0, I, J, K, R)
    Hv = oracle.gn_matvec_hv(w, v, 0.0, I, J, K, R)
    assert abs(u @ Hv - Hu @ v) <= 1e-12 * abs(u @ Hv)
    assert v @ Hv > 0
    d = oracle.jtj_diag(w, I, J, K, R)
    for j in list(range(0, n, 11)) + [n - 1]:
        e = np.zeros(n)
        e[j] = 1.0
        np.testing.assert_allclose(oracle.gn_matvec_hv(w, e, 0.0, I, J, K, R)[j], d[j], rtol=1e-13)


def test_jtj_diag_equals_explicit():
    I, J, K, R = 4, 3, 2, 3
    w = rand_w(I, J, K, R)
    Jm = jac.jacobian_entrywise(w, I, J, K, R)
    np.testing.assert_allclose(oracle.jtj_diag(w, I, J, K, R), np.sum(Jm * Jm, axis=0), rtol=1e-13)


# --------------------------------------------------------------------------- CG
def _dense_system(I, J, K, R, lam, seed=1):
    rng = np.random.default_rng(seed)
    w = rand_w(I, J, K, R, rng=rng)
    Jm = jac.jacobian_entrywise(w, I, J, K, R)
    H = Jm.T @ Jm + lam * np.eye(Jm.shape[1])
    rhs = rng.standard_normal(Jm.shape[1])
    return w, H, rhs


@pytest.mark.parametrize("jacobi", [False, True])
def test_cg_full_length_equals_dense_solve(jacobi):
    """CG terminates with the exact solution in ≤ n steps (Thm)."""
    I, J, K, R = 3, 2, 2, 2
    lam = 0.5
    w, H, rhs = _dense_system(I, J, K, R, lam)
    n = H.shape[0]
    out = oracle.cg(w, rhs, lam, 3 * n, I, J, K, R, tol=1e-26, jacobi=jacobi)
    np.testing.assert_allclose(out["x"], np.linalg.solve(H, rhs), rtol=1e-9, atol=1e-11)


def test_cg_one_iteration_closed_form():
    """x^(1) = α r^(0) with α = ‖r‖² / ⟨r, H r⟩ (Alg. CG-dGN, first pass)."""
    I, J, K, R = 4, 3, 3, 2
    lam = 1e-3
    w, H, rhs = _dense_system(I, J, K, R, lam, seed=2)
    out = oracle.cg(w, rhs, lam, 1, I, J, K, R)
    alpha = (rhs @ rhs) / (rhs @ H @ rhs)
    np.testing.assert_allclose(out["x"], alpha * rhs, rtol=1e-12)
    np.testing.assert_allclose(out["alpha"][0], alpha, rtol=1e-12)
    # Jacobi: x = M^{-1/2} α̂ r̂ with r̂ = M^{-1/2} rhs, M = diag(H)
    m = 1.0 / np.sqrt(np.diag(H))
    rh = m * rhs
    Bh = (m[:, None] * H) * m[None, :]
    ah = (rh @ rh) / (rh @ Bh @ rh)
    outj = oracle.cg(w, rhs, lam, 1, I, J, K, R, jacobi=True)
    np.testing.assert_allclose(outj["x"], m * ah * rh, rtol=1e-12)


def test_cg_zero_rhs_is_solved_by_zero():
    """Reading R33: r^(0) = 0 is solved by x^(0) = 0 = (J^T J + lam I)^{-1} 0 without iterating (the printed
    loop would form alpha = 0/0), for the plain and the Jacobi system."""
    I, J, K, R = 4, 3, 3, 2
    w, H, rhs = _dense_system(I, J, K, R, 1e-3, seed=5)
    for jacobi in (False, True):
        out = oracle.cg(w, np.zeros_like(rhs), 1e-3, 5, I, J, K, R, jacobi=jacobi)
        assert out["status"] == 0 and out["iters"] == 0
        assert np.all(out["x"] == 0.0)


def test_cg_residual_identity_and_monotone_energy():
    """ε = ‖r^(i)‖² equals ‖b − A x^(i)‖²; the A-norm error is monotone."""
    I, J, K, R = 4, 3, 3, 2
    lam = 1e-2
    w, H, rhs = _dense_system(I, J, K, R, lam, seed=3)
    out = oracle.cg(w, rhs, lam, 8, I, J, K, R, history=True)
    xs = np.linalg.solve(H, rhs)
    prev = np.inf
    for i in range(out["iters"]):
        xi = out["x_hist"][i]
        res = rhs - H @ xi
        np.testing.assert_allclose(out["r2"][i], res @ res, rtol=1e-8, atol=1e-14 * (rhs @ rhs))
        err = (xs - xi) @ H @ (xs - xi)
        assert err <= prev * (1 + 1e-12)
        prev = err


def test_cg_large_damping_limit():
    """μ → ∞: (JᵀJ + μI) x = rhs gives x → rhs / μ."""
    I, J, K, R = 4, 3, 2, 2
    w, _, rhs = _dense_system(I, J, K, R, 0.0, seed=4)
    lam = 1e9
    out = oracle.cg(w, rhs, lam, 3, I, J, K, R)
    np.testing.assert_allclose(out["x"] * lam, rhs, rtol=0, atol=1e-5 * np.abs(rhs).max())


# --------------------------------------------------------------------------- diagonal regularizer D (NEXT #1)
def _expand_damp(d, I, J, K, R):
    """Per-(mode, r) values -> the diagonal of D in w-layout (gamma_l^(r) I_{I_l})."""
    return np.concatenate([np.repeat(d[:R], I), np.repeat(d[R:2 * R], J), np.repeat(d[2 * R:], K)])


def test_reg_gamma_makes_jtj_diagonally_dominant():
    """adding gamma to the diagonal makes every row of J^T J + D dominate each of its
    off-diagonal entries: (J^T J)_ii + gamma_i >= |(J^T J)_ij| for all j (the paper's sufficient choice)."""
    for (I, J, K, R, seed) in [(4, 3, 2, 3, 0), (3, 5, 4, 2, 1), (2, 2, 2, 4, 2)]:
        rng = np.random.default_rng(seed)
        w = rng.standard_normal(R * (I + J + K)) * rng.uniform(0.2, 3.0, R * (I + J + K))
        Jm = jac.jacobian_entrywise(w, I, J, K, R)
        H = Jm.T @ Jm
        D = _expand_damp(oracle.reg_gamma(w, I, J, K, R), I, J, K, R)
        off = np.abs(H - np.diag(np.diag(H)))
        assert np.all(np.diag(H) + D >= off.max(axis=1) * (1 - 1e-12))
        # and gamma is not vacuous: without it dominance fails for these random factors
        assert not np.all(np.diag(H) >= off.max(axis=1))


def test_reg_gamma_norm_balanced_closed_form():
    """Norm-balanced factors (||X_r|| = ||Y_r|| = ||Z_r|| = a_r): gamma_l^(r) = a_r^2 max_r' a_r'^2."""
    I, J, K, R = 5, 4, 3, 3
    rng = np.random.default_rng(7)
    a = np.array([0.5, 2.0, 1.3])
    cols = []
    for n in (I, J, K):
        M = rng.standard_normal((n, R))
        cols.append(M / np.linalg.norm(M, axis=0) * a)
    w = w_of(*cols)
    g = oracle.reg_gamma(w, I, J, K, R)
    ref = a ** 2 * np.max(a ** 2)
    np.testing.assert_allclose(g, np.concatenate([ref, ref, ref]), rtol=1e-14)


@pytest.mark.parametrize("lam", [0.0, 1e-3, 0.7])
def test_damped_matvec_against_explicit(lam):
    """(J^T J + lam D) v with D = diag(gamma), Thm Hv and plain routes vs explicit."""
    I, J, K, R = 4, 3, 3, 2
    rng = np.random.default_rng(11)
    w = rng.standard_normal(R * (I + J + K))
    v = rng.standard_normal(R * (I + J + K))
    gam = oracle.reg_gamma(w, I, J, K, R)
    Jm = jac.jacobian_entrywise(w, I, J, K, R)
    ref = Jm.T @ (Jm @ v) + lam * _expand_damp(gam, I, J, K, R) * v
    np.testing.assert_allclose(oracle.gn_matvec_hv(w, v, lam, I, J, K, R, damp=gam), ref, rtol=1e-12,
                               atol=1e-13 * np.abs(ref).max())
    np.testing.assert_allclose(oracle.gn_matvec_plain(w, v, lam, I, J, K, R, damp=gam), ref, rtol=1e-12,
                               atol=1e-13 * np.abs(ref).max())


@pytest.mark.parametrize("jacobi", [False, True])
def test_damped_cg_full_length_equals_dense_solve(jacobi):
    """CG on M^{-1/2}(J^T J + mu D)M^{-1/2} with M = diag(J^T J) + mu diag(D) reaches
    the dense solution of (J^T J + mu D) x = rhs."""
    I, J, K, R = 3, 2, 2, 2
    mu = 0.3
    rng = np.random.default_rng(5)
    w = rng.standard_normal(R * (I + J + K))
    rhs = rng.standard_normal(R * (I + J + K))
    gam = oracle.reg_gamma(w, I, J, K, R)
    Jm = jac.jacobian_entrywise(w, I, J, K, R)
    H = Jm.T @ Jm + mu * np.diag(_expand_damp(gam, I, J, K, R))
    out = oracle.cg(w, rhs, mu, 60, I, J, K, R, tol=1e-26, jacobi=jacobi, damp=gam)
    np.testing.assert_allclose(out["x"], np.linalg.solve(H, rhs), rtol=1e-9, atol=1e-11)
    # with Jacobi the preconditioned diagonal is exactly 1 (first step: alpha uses B_ii = 1)
    if jacobi:
        m = 1.0 / np.sqrt(np.diag(H))
        np.testing.assert_allclose((m[:, None] * H * m[None, :]).diagonal(), 1.0, rtol=1e-14)


# --------------------------------------------------------------------------- dGN outer loop (NEXT #2)
def test_cg_budget_interval():
    """cg_maxiter at dGN iteration k is drawn from [1 + ceil(k^0.4), 2 + ceil(k^0.9)]."""
    import synth
    b = synth.cg_budget(200, seed=3)
    ks = np.arange(1, 201)
    assert np.all(b >= 1 + np.ceil(ks ** 0.4)) and np.all(b <= 2 + np.ceil(ks ** 0.9))
    assert b[-1] <= 120 and b[0] in (2, 3)


def test_linearized_model_matches_gradient_form():
    """1/2||f + J x||^2 = F + <grad F, x> + 1/2 x^T J^T J x (gain-ratio denominator),
    checked with the explicit Jacobian; the oracle's dGN evaluates the left side entry by entry."""
    I, J, K, R = 4, 3, 2, 2
    rng = np.random.default_rng(21)
    T = rng.standard_normal(I * J * K)
    w = rng.standard_normal(R * (I + J + K))
    x = 0.3 * rng.standard_normal(R * (I + J + K))
    Jm = jac.jacobian_entrywise(w, I, J, K, R)
    r = jac.residual(T, w, I, J, K, R)
    f, g = oracle.cpd_eval(T, w, I, J, K, R)
    lhs = 0.5 * np.sum((r + Jm @ x) ** 2)
    rhs_ = f + g @ x + 0.5 * x @ (Jm.T @ (Jm @ x))
    assert abs(lhs - rhs_) <= 1e-12 * abs(lhs)


def _exact_problem(I, J, K, R, seed):
    rng = np.random.default_rng(seed)
    A, B, C = (rng.standard_normal((n, R)) for n in (I, J, K))
    t = build_T(A, B, C)
    w0 = rng.standard_normal(R * (I + J + K))
    return dense_T(t), w0


def test_dgn_converges_on_exact_rank_tensor():
    """From a random start the full dGN iteration (gamma damping, Jacobi CG, norm balancing, random CG budget)
    drives the relative error of an exactly rank-3 tensor below tol (stopping condition 1)."""
    import synth
    I, J, K, R = 9, 8, 7, 3
    T, w0 = _exact_problem(I, J, K, R, 5)
    out = oracle.dgn(T, w0, I, J, K, R, synth.cg_budget(200, seed=1), tol=1e-6)
    assert out["reason"] == 1, out
    assert out["hist"][-1, 1] < 1e-6


def test_dgn_damping_rule_and_balancing():
    """mu^(0) = mean|T| (tau = 1); g < 0.25 -> 3 mu, g > 0.75 -> mu / 3;
    norm balancing leaves the tensor (hence F) unchanged and equalises the column norms."""
    import synth
    I, J, K, R = 6, 5, 4, 3
    T, w0 = _exact_problem(I, J, K, R, 9)
    T = T + 0.05 * np.random.default_rng(1).standard_normal(T.size)
    cgi = synth.cg_budget(12, seed=2)
    out = oracle.dgn(T, w0, I, J, K, R, cgi, maxiter=12, tol=0.0)
    h = out["hist"]
    assert abs(h[0, 2] - np.mean(np.abs(T))) <= 1e-15 * h[0, 2]
    for k in range(len(h) - 1):
        g, mu, mun = h[k, 3], h[k, 2], h[k + 1, 2]
        want = 3 * mu if g < 0.25 else (mu / 3 if g > 0.75 else mu)
        assert abs(mun - want) <= 1e-14 * want
    # balancing: same F trajectory for the first step with and without it; balanced norms are equal
    nb = oracle.dgn(T, w0, I, J, K, R, cgi, maxiter=1, tol=0.0, balance=False)
    bb = oracle.dgn(T, w0, I, J, K, R, cgi, maxiter=1, tol=0.0, balance=True)
    assert abs(nb["hist"][0, 0] - bb["hist"][0, 0]) <= 1e-12 * nb["hist"][0, 0]
    A, B, C = jac.factors_from_w(bb["w"], I, J, K, R)
    na, nb_, nc = (np.linalg.norm(M, axis=0) for M in (A, B, C))
    np.testing.assert_allclose(na, nb_, rtol=1e-13)
    np.testing.assert_allclose(na, nc, rtol=1e-13)


# --------------------------------------------------------------------------- gamma: the per-mode pairing
def _tight_factors(norms, I, J, K, seed):
    """Columns nearly parallel to e_0 (1e-3 perturbation) with prescribed norms norms[l][r]: every Cauchy-Schwarz
    bound behind gamma is then attained to 1e-3, so the dominance rows are tight."""
    rng = np.random.default_rng(seed)
    out = []
    for l, n in enumerate((I, J, K)):
        cols = []
        for r in range(len(norms[l])):
            v = np.zeros(n)
            v[0] = 1.0
            v += 1e-3 * rng.standard_normal(n)
            cols.append(norms[l][r] * v / np.linalg.norm(v))
        out.append(np.stack(cols, axis=1))
    return out


def _dominant(H, d):
    off = np.abs(H - np.diag(np.diag(H))).max(axis=1)
    return bool(np.all(np.diag(H) + d >= off * (1 - 1e-12)))


def test_reg_gamma_pairing_is_the_one_that_dominates():
    """gamma_X^(r) = ||Y_r|| ||Z_r|| M, gamma_Y^(r) = ||X_r|| ||Z_r|| M, gamma_Z^(r) = ||X_r|| ||Y_r|| M with
    M = max over r' of all three products. On factors whose columns are nearly parallel
    (the off-diagonal entries of J^T J attain their Cauchy-Schwarz bounds) with column r of mode r much
    shorter than the rest, every row of J^T J + D dominates each of its off-diagonal entries with the oracle's
    gamma. The test also shows it discriminates: every other pairing of the three products to the modes, and
    M taken over a single product, break dominance on at least one of the three cyclic variants."""
    import itertools
    I, J, K, R = 3, 4, 3, 3
    base = np.array([[0.05, 2.0, 3.0], [1.5, 0.04, 2.5], [2.2, 1.7, 0.06]])
    configs = [np.roll(base, s, axis=0) for s in range(3)]   # which product attains M rotates too
    wrong_pairings = set(p for p in itertools.permutations(("YZ", "XZ", "XY")) if p != ("YZ", "XZ", "XY"))
    broken_pairings, broken_partial_max = set(), set()
    for ci, nm in enumerate(configs):
        X, Y, Z = _tight_factors(nm, I, J, K, seed=ci)
        w = w_of(X, Y, Z)
        Jm = jac.jacobian_entrywise(w, I, J, K, R)
        H = Jm.T @ Jm
        gam = oracle.reg_gamma(w, I, J, K, R)
        assert _dominant(H, _expand_damp(gam, I, J, K, R)), ci
        # negative controls (mutations of the rule, written here only to show the pin discriminates)
        nx, ny, nz = (np.linalg.norm(F, axis=0) for F in (X, Y, Z))
        prods = {"YZ": ny * nz, "XZ": nx * nz, "XY": nx * ny}
        Mx = max(p.max() for p in prods.values())
        for perm in wrong_pairings:
            if not _dominant(H, _expand_damp(np.concatenate([prods[p] * Mx for p in perm]), I, J, K, R)):
                broken_pairings.add(perm)
        for key in prods:
            g1 = np.concatenate([prods[p] * prods[key].max() for p in ("YZ", "XZ", "XY")])
            if not _dominant(H, _expand_damp(g1, I, J, K, R)):
                broken_partial_max.add(key)
    assert broken_pairings == wrong_pairings
    assert broken_partial_max == {"YZ", "XZ", "XY"}


# --------------------------------------------------------------------------- dGN: stopping rule and gain ratio
def test_dgn_stop_rule_constructed_histories():
    """The stopping conditions of PAPER.md:2756-2773 on constructed histories, each made to hold while every
    earlier condition fails (readings R20, R21): the rule returns that condition, and moving the history just
    across its threshold (10% either side) turns it off. maxiter = 15 -> c = 1 + ceil(15/10) = 3, so 5 and 6
    are checked at k = 9, 12, ... (k > 2c, k = 0 mod c) over the windows [k-6, k-3) and [k-3, k)."""
    S = oracle.dgn_stop
    tol, nT2, mx = 1e-4, 4.0, 15
    big = 1.0
    lo, hi = 0.9 * tol, 1.1 * tol
    # 1: relative error below tol
    assert S(1, [0.5, lo], mx, tol, big, big, nT2) == 1
    assert S(1, [0.5, hi], mx, tol, big, big, nT2) == 0
    # 2: step below tol (the error did not change either: 2 is checked before 3)
    assert S(1, [0.5, 0.5], mx, tol, lo, big, nT2) == 2
    assert S(1, [0.5, 0.3], mx, tol, hi, big, nT2) == 0
    # 3: improvement of the relative error below tol
    assert S(1, [0.5, 0.5 - lo], mx, tol, big, big, nT2) == 3
    assert S(1, [0.5, 0.5 - hi], mx, tol, big, big, nT2) == 0
    # 4: infinity norm of the gradient below tol
    assert S(1, [0.5, 0.3], mx, tol, big, lo, nT2) == 4
    assert S(1, [0.5, 0.3], mx, tol, big, hi, nT2) == 0
    # 5: mean of rel over [3, 6) minus mean over [6, 9) below tol (oscillation without decrease), at k = 9:
    #    rel[3..5] = 0.6, 0.7, 0.6 and rel[6..8] = 0.7, 0.6, 0.6 + 3 lo: m1 - m2 = -lo < tol; rel[9] = 0.65
    rel5 = [1.0, 0.9, 0.8, 0.6, 0.7, 0.6, 0.7, 0.6, 0.6 + 3 * lo, 0.65]
    assert S(9, rel5, mx, tol, big, big, nT2) == 5
    assert S(8, rel5, mx, tol, big, big, nT2) == 0            # only checked at k = 0 mod c
    assert S(6, rel5[:7], mx, tol, big, big, nT2) == 0        # ... and k > 2c
    rel5b = list(rel5)
    rel5b[8] = 0.6 - 3 * hi                                   # m1 - m2 = 1.1 tol
    assert S(9, rel5b, mx, tol, big, big, nT2) == 0
    # 6: mean improvement over [6, 9) below 1e-3 of the mean error (decreasing, so 5 fails): steps of d with
    #    3 d = ... rel[6..9] = 0.5, 0.5 - d, 0.5 - 2d, 0.5 - 3d; imp = d vs 1e-3 m2 = 1e-3 (0.5 - d)
    def rel6(d):
        return [1.0, 0.9, 0.8, 0.7, 0.6, 0.55, 0.5, 0.5 - d, 0.5 - 2 * d, 0.5 - 3 * d]
    thr = 1e-3 * 0.5 / (1 + 1e-3)                           # d = 1e-3 (0.5 - d)
    assert S(9, rel6(0.9 * thr), mx, tol, big, big, nT2) == 6
    assert S(9, rel6(1.1 * thr), mx, tol, big, big, nT2) == 0
    # 7: divergence: rel > max(1, ||T||^2) / (1e-16 + tol) = 4 / 1e-4 = 4e4
    assert S(1, [3e4, 1.1 * 4e4], mx, tol, big, big, nT2) == 7
    assert S(1, [3e4, 0.9 * 4e4], mx, tol, big, big, nT2) == 0
    assert S(1, [0.5, 2.2], mx, 0.5, big, big, 0.25) == 7      # max(1, ||T||^2) = 1: threshold 1 / 0.5 = 2
    assert S(1, [0.5, 1.8], mx, 0.5, big, big, 0.25) == 0


def _small_problem(I, J, K, R, seed, sigma, scale=1.0):
    rng = np.random.default_rng(seed)
    A, B, C = (rng.standard_normal((n, R)) for n in (I, J, K))
    t = scale * (build_T(A, B, C) + sigma * rng.standard_normal((I, J, K)))
    return dense_T(t), rng


def test_dgn_stops_in_runs():
    """Runs of the oracle's dGN loop that must stop with a given condition at k = 1:
    * 2 (step): w0 = 0 is a stationary point (every MTTKRP and W Pi vanish), so -grad F = 0 and CG returns x = 0
      (reading R33): ||x|| = 0 < tol while the relative error is 1 (3 holds too, but 2 comes first).
    * 4 (gradient): T and w0 scaled by s and s^(1/3) (s = 1e-9): the relative error and its first improvement
      are scale-free (large), the step scales as s^(1/3) = 1e-3 > tol, the gradient as s^(5/3) < tol.
    * 7 (divergence): ||T|| < 1 and w0 huge: after one Gauss-Newton step the model is still far worse than
      0, rel > 1 / (1e-16 + tol) with tol = 1 (and the step, improvement and gradient are all > 1).
    Each is checked on the oracle's own history and on the final w with the pinned evaluation."""
    I, J, K, R = 5, 4, 3, 2
    T, rng = _small_problem(I, J, K, R, 31, 0.1)
    nT = float(np.linalg.norm(T))
    cgi = np.full(5, 4, dtype=np.int32)
    # 2
    out = oracle.dgn(T, np.zeros(R * (I + J + K)), I, J, K, R, cgi, maxiter=5, tol=1e-8, use_gamma=False,
                     jacobi=False)
    assert out["reason"] == 2 and out["iters"] == 1, out
    assert out["hist"][0, 4] == 0.0 and abs(out["hist"][0, 1] - 1.0) < 1e-15
    # 4
    s = 1e-9
    Ts = T * s
    w0 = rng.standard_normal(R * (I + J + K)) * s ** (1 / 3)
    out = oracle.dgn(Ts, w0, I, J, K, R, cgi, maxiter=5, tol=1e-4)
    assert out["reason"] == 4 and out["iters"] == 1, out
    f0, _ = oracle.cpd_eval(Ts, w0, I, J, K, R)
    f1, g1 = oracle.cpd_eval(Ts, out["w"], I, J, K, R)
    rel0, rel1 = math.sqrt(2 * f0) / (nT * s), math.sqrt(2 * f1) / (nT * s)
    assert rel1 >= 1e-4 and abs(rel0 - rel1) >= 1e-4 and out["hist"][0, 4] >= 1e-4
    assert np.abs(g1).max() < 1e-4
    # 7
    Tt = T / (2 * nT)                       # ||T|| = 1/2
    w0 = 30.0 * rng.standard_normal(R * (I + J + K))
    out = oracle.dgn(Tt, w0, I, J, K, R, cgi, maxiter=5, tol=1.0)
    assert out["reason"] == 7 and out["iters"] == 1, out
    f1, g1 = oracle.cpd_eval(Tt, out["w"], I, J, K, R)
    assert math.sqrt(2 * f1) / 0.5 > 1.0 and np.abs(g1).max() >= 1.0 and out["hist"][0, 4] >= 1.0


def test_dgn_gain_ratio_against_explicit_jacobian():
    """The gain ratio of one dGN step (reading R19): g = (F(w0) - F(w1)) /
    (F(w0) - 1/2 ||f(w0) + J_f(w0) x||^2) with x = w1 - w0 (no balancing), recomputed with the explicit
    Jacobian of Lemma partialf and the pinned evaluation, equals the oracle's recorded g."""
    I, J, K, R = 4, 3, 3, 2
    T, rng = _small_problem(I, J, K, R, 41, 0.3)
    w0 = rng.standard_normal(R * (I + J + K))
    for jacobi in (False, True):
        out = oracle.dgn(T, w0, I, J, K, R, np.array([3], dtype=np.int32), maxiter=1, tol=0.0, balance=False,
                         jacobi=jacobi)
        x = out["w"] - w0
        f0, _ = oracle.cpd_eval(T, w0, I, J, K, R)
        f1, _ = oracle.cpd_eval(T, out["w"], I, J, K, R)
        Jm = jac.jacobian_entrywise(w0, I, J, K, R)
        r0 = jac.residual(T, w0, I, J, K, R)
        g = (f0 - f1) / (f0 - 0.5 * np.sum((r0 + Jm @ x) ** 2))
        assert abs(out["hist"][0, 3] - g) <= 1e-10 * abs(g), (out["hist"][0, 3], g)
        assert abs(out["hist"][0, 0] - f1) <= 1e-14 * f1
