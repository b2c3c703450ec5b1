"""Pins of the MLSVD / compression oracle (oracle/mlsvd.py) to what the paper and mathematics fix.

Values the paper prints for the warming-up tensor (tests/golden/warmup_mlsvd.json, cited there),
theorems about the MLSVD (De Lathauwer et al.), the L=2 special case that
reduces to a library SVD, and exact identities on tensors of known multilinear rank.
"""
import json
import math
import os

import numpy as np
import pytest

from oracle import jacobian as jac
from oracle import mlsvd as M

RNG = np.random.default_rng(2110_05997)


def warmup_T(golden_dir):
    """t_ijk = φ(x_i, y_j, z_k) on the printed grids (R16: z = k/3)."""
    g = json.load(open(os.path.join(golden_dir, "warmup.json")))
    x, y = np.array(g["x"]), np.array(g["y"])
    z = np.array(g["z_num"], dtype=np.float64) / g["z_den"]
    X, Y, Z = np.meshgrid(x, y, z, indexing="ij")
    t = (np.cos(1 - X) * np.sin(1 + Y ** 2) - np.sin(1 + X ** 2) * np.exp(X ** 2 + Y ** 2 + Z ** 2)
         - np.cos(X) * np.log(1 + Z))
    return t, jac.storage_from_tensor(t)


@pytest.fixture(scope="module")
def golden(golden_dir):
    return json.load(open(os.path.join(golden_dir, "warmup_mlsvd.json")))


def test_table_4_5_truncation_errors(golden_dir, golden):
    """Table 4.5: all 27 truncations of the 3×3×3 core, 8 printed decimals."""
    _, T = warmup_T(golden_dir)
    m = M.mlsvd(T, 6, 5, 4, 3)
    assert m["P"] == (3, 3, 3)
    for shape, printed in golden["table_4_5"]:
        e = M.truncation_error(m["S"], shape)
        assert abs(e - printed) <= 0.5e-8 + 1e-12, (shape, e, printed)


def test_printed_core_magnitudes(golden_dir, golden):
    """The printed core, frontal slices, to one unit of its last printed digit.
    Signs of singular vectors are not fixed by the paper (reading R23): magnitudes only."""
    _, T = warmup_T(golden_dir)
    S = M.mlsvd(T, 6, 5, 4, 3)["S"]
    for k, slab in enumerate(golden["core_frontal_slices"]):
        for a, row in enumerate(slab):
            for b, v in enumerate(row):
                s = repr(abs(v))
                dec = len(s.split(".")[1]) if "." in s else 0
                assert abs(abs(S[a, b, k]) - abs(v)) <= 10.0 ** (-dec) + 1e-12, (a, b, k, S[a, b, k], v)


def test_full_mlsvd_truncates_to_3x3x3_exactly(golden_dir, golden):
    """The full MLSVD (P_l = I_l) truncated to 3×3×3 has relative error ~1e-14 (printed 3.85e-14,
    PAPER.md:2926): the warming-up tensor has multilinear rank (3, 3, 3); and Alg. Compression picks
    exactly those ranks."""
    _, T = warmup_T(golden_dir)
    m = M.mlsvd(T, 6, 5, 4, 100)
    assert m["P"] == (6, 5, 4)
    e = M.truncation_error(m["S"], (3, 3, 3))
    assert e < 1e-12 and e > 0.0, e
    assert abs(math.log10(e) - math.log10(golden["truncation_error_3x3x3"])) < 1.5
    c = M.compress(T, 6, 5, 4, 100, 1e-6)
    assert c["ranks"] == (3, 3, 3)
    # with a loose tolerance the ranks shrink, and the guarantee of Alg. Compression holds
    c2 = M.compress(T, 6, 5, 4, 100, 1e-2)
    assert max(c2["ranks"]) < 3
    assert M.truncation_error(m["S"], c2["ranks"]) ** 2 < 1e-2


def test_energy_initialisation(golden_dir, golden):
    """MLSVD-energy initialisation: picks s111, s212, s122 (45.84, 1.12, 1.48)
    and the initial CPD has relative error 0.0153."""
    t, T = warmup_T(golden_dir)
    m = M.mlsvd(T, 6, 5, 4, 3)
    W1, W2, W3, picks = M.energy_init(m["S"], 3)
    assert sorted(tuple(p + 1 for p in pk) for pk in picks) == sorted(tuple(p) for p in golden["init_multi_indexes_1based"])
    vals = sorted(abs(m["S"][p]) for p in picks)
    assert np.allclose(vals, sorted(golden["init_values"]), atol=0.01)
    A, B, C = M.uncompress(m["U"], [W1, W2, W3])
    rec = np.einsum("ir,jr,kr->ijk", A, B, C)
    err = np.linalg.norm(t - rec) / np.linalg.norm(t)
    # printed 0.0153 is the value cut (not rounded) to 4 decimals: 0.0153 <= err < 0.0154
    assert golden["init_rel_error"] <= err < golden["init_rel_error"] + 1e-4, err


@pytest.mark.parametrize("dims", [(5, 4, 3), (3, 6, 4), (7, 2, 5)])
def test_mlsvd_theorem_properties(dims):
    """Thm MLSVD and Thm MLSVD-properties item 4 (1378-1386) for the full MLSVD:
    T = (U1, U2, U3)·S, orthonormal U_l, all-orthogonality of the hyperslices of S, their norms are
    the sigma's in decreasing order, and ||T||² = sum sigma_r^(l)² for every mode."""
    I, J, K = dims
    t = RNG.standard_normal(dims)
    T = jac.storage_from_tensor(t)
    m = M.mlsvd(T, I, J, K, 1000)
    U1, U2, U3 = m["U"]
    S = m["S"]
    for U in m["U"]:
        assert np.allclose(U.T @ U, np.eye(U.shape[1]), atol=1e-13)
    rec = np.einsum("ai,bj,ck,ijk->abc", U1, U2, U3, S)
    assert np.allclose(rec, t, atol=1e-13)
    nT2 = float(np.sum(t * t))
    for l in range(3):
        Sl = jac.unfold(S, l + 1)
        Gs = Sl @ Sl.T
        off = Gs - np.diag(np.diag(Gs))
        assert np.abs(off).max() <= 1e-12 * nT2
        assert np.allclose(np.sqrt(np.diag(Gs)), m["sigma"][l], rtol=1e-12, atol=1e-12)
        assert np.all(np.diff(m["sigma"][l]) <= 1e-12)
        assert abs(np.sum(m["sigma"][l] ** 2) - nT2) <= 1e-12 * nT2


def test_two_way_case_is_the_svd():
    """For L = 2 the MLSVD is the SVD: a K = 1 tensor is the matrix M = T_::1; its
    mode-1 singular values / vectors equal numpy's SVD of M (LAPACK gesdd, an independent routine)."""
    I, J = 7, 5
    Mx = RNG.standard_normal((I, J))
    T = jac.storage_from_tensor(Mx[:, :, None])
    m = M.mlsvd(T, I, J, 1, 100)
    Us, s, Vt = np.linalg.svd(Mx, full_matrices=False)
    assert np.allclose(m["sigma"][0][:J], s, rtol=1e-12)
    assert np.allclose(m["sigma"][1], s, rtol=1e-12)
    for c in range(J):
        assert abs(abs(m["U"][0][:, c] @ Us[:, c]) - 1.0) < 1e-12
        assert abs(abs(m["U"][1][:, c] @ Vt[c]) - 1.0) < 1e-12
    # Thm SVD-truncation: ||M - M~||² = sum of the dropped sigma²
    for r in range(1, J):
        Mt = m["U"][0][:, :r] @ np.diag(m["S"][:r, :r, 0].diagonal()) @ m["U"][1][:, :r].T
        assert abs(np.linalg.norm(Mx - Mt) ** 2 - np.sum(s[r:] ** 2)) <= 1e-12 * np.sum(s ** 2)


def test_core_by_unfolding_formula_equals_multilinear_definition():
    """S by Thm unfolding-formula (U1^T T_(1) (U3 ⊗ U2)) equals the entrywise
    multilinear multiplication; and the Gram entries by hyperslice inner products equal T_(l)T_(l)^T."""
    I, J, K = 5, 4, 6
    t = RNG.standard_normal((I, J, K))
    T = jac.storage_from_tensor(t)
    m = M.mlsvd(T, I, J, K, 3)
    U1, U2, U3 = m["U"]
    S2 = M.core_unfolding(T, I, J, K, U1, U2, U3)
    assert np.allclose(m["S"], S2, atol=1e-13)
    for mode, n in ((1, I), (2, J), (3, K)):
        G = M.unfolding_gram(T, I, J, K, mode)
        for p in range(n):
            for q in range(n):
                assert abs(M.gram_entry(T, I, J, K, mode, p, q) - G[p, q]) <= 1e-13 * abs(G).max()


def test_exact_multilinear_rank_and_compressed_cpd():
    """T = (M1, M2, M3)·G with a random (2,3,4) core has multilinear rank (2,3,4) (Thm MLSVD-properties
    item 1): sigma^(l)_k = 0 beyond it and Alg. Compression returns those ranks with ~0 error.
    Remark mlsvd-cpd: for T = [[A,B,C]], the core is [[U1^T A, U2^T B, U3^T C]]
    and uncompressing those factors returns A, B, C."""
    I, J, K = 9, 8, 7
    G = RNG.standard_normal((2, 3, 4))
    M1, M2, M3 = (RNG.standard_normal((n, r)) for n, r in ((I, 2), (J, 3), (K, 4)))
    t = np.einsum("ia,jb,kc,abc->ijk", M1, M2, M3, G)
    T = jac.storage_from_tensor(t)
    m = M.mlsvd(T, I, J, K, 6)
    nT = np.linalg.norm(t)
    for l, r in enumerate((2, 3, 4)):
        assert np.all(m["sigma"][l][r:] <= 1e-6 * nT)   # sqrt of a ~u·||T||² eigenvalue
        assert m["sigma"][l][r - 1] > 1e-3 * nT
    c = M.compress(T, I, J, K, 6, 1e-10)
    assert c["ranks"] == (2, 3, 4)
    rec = np.einsum("ia,jb,kc,abc->ijk", *c["U"], c["S"])
    assert np.linalg.norm(rec - t) <= 1e-12 * nT
    R = 3
    A, B, C = (RNG.standard_normal((n, R)) for n in (I, J, K))
    t = np.einsum("ir,jr,kr->ijk", A, B, C)
    T = jac.storage_from_tensor(t)
    c = M.compress(T, I, J, K, R, 1e-12)
    assert c["ranks"] == (3, 3, 3)
    Ws = [U.T @ X for U, X in zip(c["U"], (A, B, C))]
    assert np.allclose(c["S"], np.einsum("ar,br,cr->abc", *Ws), atol=1e-12 * np.linalg.norm(t))
    for X, Xr in zip((A, B, C), M.uncompress(c["U"], Ws)):
        assert np.allclose(X, Xr, atol=1e-12 * np.abs(X).max())


def test_energy_bound_of_truncation():
    """Thm energy-mlsvd: ||T - T~||² <= sum_l sum_{r > R~_l} sigma_r^(l)²,
    on a noisy low-rank tensor, for several truncation shapes (full MLSVD)."""
    I, J, K = 8, 7, 6
    A, B, C = (RNG.standard_normal((n, 3)) for n in (I, J, K))
    t = np.einsum("ir,jr,kr->ijk", A, B, C) + 0.05 * RNG.standard_normal((I, J, K))
    T = jac.storage_from_tensor(t)
    m = M.mlsvd(T, I, J, K, 100)
    for shape in [(1, 1, 1), (2, 3, 2), (3, 3, 3), (5, 2, 6)]:
        Ut = [m["U"][l][:, :shape[l]] for l in range(3)]
        St = m["S"][:shape[0], :shape[1], :shape[2]]
        rec = np.einsum("ia,jb,kc,abc->ijk", *Ut, St)
        lhs = np.linalg.norm(t - rec) ** 2
        rhs = sum(np.sum(m["sigma"][l][shape[l]:] ** 2) for l in range(3))
        assert lhs <= rhs * (1 + 1e-12) + 1e-20
        # and the orthogonal projection identity ||T - T~|| = ||S - S~|| (PAPER.md:2553 footnote)
        assert abs(math.sqrt(lhs) / np.linalg.norm(t) - M.truncation_error(m["S"], shape)) < 1e-12


def test_normalize_cpd_output_form():
    """The unit-column output form: sum_r lambda_r w_r^(1)⊗w_r^(2)⊗w_r^(3) is the same
    tensor, every column has unit norm, lambda_r = prod of the column norms; a zero column gives lambda 0."""
    A, B, C = (RNG.standard_normal((n, 4)) for n in (5, 6, 7))
    C[:, 2] = 0.0
    (a, b, c), lam = M.normalize_cpd([A, B, C])
    t0 = np.einsum("ir,jr,kr->ijk", A, B, C)
    t1 = np.einsum("r,ir,jr,kr->ijk", lam, a, b, c)
    assert np.allclose(t0, t1, atol=1e-13)
    for X in (a, b):
        assert np.allclose(np.linalg.norm(X, axis=0), 1.0)
    assert lam[2] == 0.0 and np.allclose(np.linalg.norm(c[:, [0, 1, 3]], axis=0), 1.0)
    assert np.allclose(lam[[0, 1, 3]], [np.linalg.norm(A[:, r]) * np.linalg.norm(B[:, r]) * np.linalg.norm(C[:, r])
                                       for r in (0, 1, 3)])


def test_st_mlsvd_error_identity_and_special_cases(golden_dir):
    """Alg. ST-MLSVD. (i) Its first step is the classic mode-1 SVD. (ii) Without
    truncation it is exact: T = (U1, U2, U3)·S. (iii) The ST-HOSVD error identity (the projections are
    orthogonal and nested): ||T - T~||^2 = sum over steps of the discarded squared singular values of that
    step. (iv) On an exactly multilinear-rank-(2,3,4) tensor it recovers the ranks with ~0 error, and on the
    warming-up tensor it gives the 3x3x3 core of the classic MLSVD up to signs (no truncation happens)."""
    I, J, K = 8, 7, 6
    A, B, C = (RNG.standard_normal((n, 3)) for n in (I, J, K))
    t = np.einsum("ir,jr,kr->ijk", A, B, C) + 0.05 * RNG.standard_normal((I, J, K))
    T = jac.storage_from_tensor(t)
    st = M.st_mlsvd(T, I, J, K, 100, 1e-3)
    cl = M.mlsvd(T, I, J, K, 100)
    assert np.allclose(st["sigma"][0], cl["sigma"][0], rtol=1e-12)
    rec = np.einsum("ia,jb,kc,abc->ijk", *st["U"], st["S"])
    lhs = np.linalg.norm(t - rec) ** 2
    rhs = sum(np.sum(st["sigma"][l][st["ranks"][l]:] ** 2) for l in range(3))
    assert abs(lhs - rhs) <= 1e-10 * np.sum(t * t), (lhs, rhs)
    assert max(st["ranks"]) < 6            # something was truncated (the identity is not vacuous)
    full = M.st_mlsvd(T, I, J, K, 100, 1e-300)
    assert full["ranks"] == (I, J, K)
    assert np.allclose(np.einsum("ia,jb,kc,abc->ijk", *full["U"], full["S"]), t, atol=1e-12)
    G = RNG.standard_normal((2, 3, 4))
    M1, M2, M3 = (RNG.standard_normal((n, r)) for n, r in ((I, 2), (J, 3), (K, 4)))
    t2 = np.einsum("ia,jb,kc,abc->ijk", M1, M2, M3, G)
    s2 = M.st_mlsvd(jac.storage_from_tensor(t2), I, J, K, 6, 1e-10)
    assert s2["ranks"] == (2, 3, 4)
    assert np.linalg.norm(np.einsum("ia,jb,kc,abc->ijk", *s2["U"], s2["S"]) - t2) <= 1e-12 * np.linalg.norm(t2)
    _, Tw = warmup_T(golden_dir)
    sw = M.st_mlsvd(Tw, 6, 5, 4, 3, 1e-6)
    cw = M.mlsvd(Tw, 6, 5, 4, 3)
    assert sw["ranks"] == (3, 3, 3)
    assert np.allclose(np.abs(sw["S"]), np.abs(cw["S"]), atol=1e-10)



@pytest.mark.parametrize("mlsvd_tol,ranks", [(3e-2, (3, 3, 3)), (6e-2, (2, 2, 2)), (1e-3, (4, 4, 3))])
def test_st_mlsvd_per_step_threshold(mlsvd_tol, ranks):
    """Alg. ST-MLSVD's per-step truncation (PAPER.md:1430-1439 with Alg. Compression's rule, 2566-2583, reading
    R32): each step keeps the smallest i with tail/total < mlsvd_tol / L, L = 3, of THAT step's singular values.
    The tensor is (Q1, Q2, Q3)·S for random orthogonal Q_l and a core of four rank-one terms s_t e_a⊗e_b⊗e_c,
    (a,b,c; s²) = (0,0,0; 1), (1,1,1; 0.6), (2,2,2; 0.02), (3,3,1; 0.005), whose mode-l unfolding rows share no
    columns: the mode-l singular values are exactly the square roots of the row sums of s², so the ranks are
    derived by hand (P_l = min(5, R = 5) = 5):
      mode 1: σ² = 1, 0.6, 0.02, 0.005, 0 (total 1.625); tail after i = 2: 0.025/1.625 = 0.01538, after i = 3:
              0.005/1.625 = 0.003077, after i = 4: 0.
      tol 3e-2 -> threshold 1e-2 -> R~1 = 3; step 1 drops term 4, so step 2 sees σ² = 1, 0.6, 0.02 (tail after
              2: 0.02/1.62 = 0.0123 >= 1e-2) -> 3, step 3 the same -> (3, 3, 3).
      tol 6e-2 -> threshold 2e-2 -> R~1 = 2; steps 2 and 3 see 1, 0.6 (tail after 1: 0.375) -> (2, 2, 2).
      tol 1e-3 -> threshold 3.33e-4 -> R~1 = 4 (tail after 3 = 0.003077); step 2 sees 1, 0.6, 0.02, 0.005 -> 4;
              step 3's rows are 1, 0.605 (terms 2 and 4 share c = 1), 0.02 -> tail after 2 = 0.0123, after 3 = 0
              -> 3: (4, 4, 3).
    A threshold of mlsvd_tol (no 1/L) or 3·mlsvd_tol gives R~1 = 2 in the first case; mlsvd_tol / 9 gives 4 in
    the second. The truncation error equals the dropped energy (ST-HOSVD identity), below mlsvd_tol."""
    n, R = 5, 5
    terms = [((0, 0, 0), 1.0), ((1, 1, 1), 0.6), ((2, 2, 2), 0.02), ((3, 3, 1), 0.005)]
    S = np.zeros((n, n, n))
    for (a, b, c), s2 in terms:
        S[a, b, c] = math.sqrt(s2)
    rng = np.random.default_rng(17)
    Q = [np.linalg.qr(rng.standard_normal((n, n)))[0] for _ in range(3)]
    t = np.einsum("ia,jb,kc,abc->ijk", Q[0], Q[1], Q[2], S)
    st = M.st_mlsvd(jac.storage_from_tensor(t), n, n, n, R, mlsvd_tol)
    assert st["ranks"] == ranks
    # step 1's singular values are the hand-derived ones
    assert np.allclose(st["sigma"][0] ** 2, [1.0, 0.6, 0.02, 0.005, 0.0], atol=1e-14)
    rec = np.einsum("ia,jb,kc,abc->ijk", *st["U"], st["S"])
    dropped = {(3, 3, 3): 0.005, (2, 2, 2): 0.025, (4, 4, 3): 0.0}[ranks]
    assert abs(np.linalg.norm(t - rec) ** 2 - dropped) <= 1e-13
    assert dropped / 1.625 < mlsvd_tol
