"""Pins of the CP-ALS oracle (oracle/als.py) to the mathematics of Alg. ALS.

Each update solves a linear least-squares problem exactly, so (i) the block of ∇F (oracle.cpd_eval, itself
pinned) of the updated mode vanishes, (ii) it equals numpy.linalg.lstsq on the materialised system
min ‖T_(l) − W (⊙)^T‖, (iii) F never increases, and (iv) the true factors of an exact-rank tensor are a
fixed point.
"""
import numpy as np
import pytest

import oracle
from oracle import als as ALS
from oracle import jacobian as jac

RNG = np.random.default_rng(1719)


def noisy(I, J, K, R, sigma, seed):
    rng = np.random.default_rng(seed)
    A, B, C = (rng.standard_normal((n, R)) for n in (I, J, K))
    t = np.einsum("ir,jr,kr->ijk", A, B, C) + sigma * rng.standard_normal((I, J, K))
    return jac.storage_from_tensor(t), (A, B, C)


@pytest.mark.parametrize("mode", [1, 2, 3])
def test_update_is_least_squares_optimal(mode):
    I, J, K, R = 7, 6, 5, 3
    T, _ = noisy(I, J, K, R, 0.3, mode)
    Ws = [RNG.standard_normal((n, R)) for n in (I, J, K)]
    new = ALS.als_update(T, Ws, mode, I, J, K)
    w = ALS._pack(new)
    _, g = oracle.cpd_eval(T, w, I, J, K, R)
    offs = [0, I * R, (I + J) * R, (I + J + K) * R]
    blk = g[offs[mode - 1]:offs[mode]]
    assert np.linalg.norm(blk) <= 1e-10 * np.linalg.norm(g[:offs[1]] if mode != 1 else g) + 1e-12
    # the other blocks are generally not zero (the test can fail)
    others = np.concatenate([g[offs[m - 1]:offs[m]] for m in (1, 2, 3) if m != mode])
    assert np.linalg.norm(others) > 1e-3


@pytest.mark.parametrize("mode", [1, 2, 3])
def test_update_equals_lstsq(mode):
    I, J, K, R = 6, 5, 4, 2
    T, _ = noisy(I, J, K, R, 0.2, 10 + mode)
    Ws = [RNG.standard_normal((n, R)) for n in (I, J, K)]
    new = ALS.als_update(T, Ws, mode, I, J, K)
    t = jac.tensor_from_storage(T, I, J, K)
    A, B, C = Ws
    KR = {1: jac.khatri_rao(C, B), 2: jac.khatri_rao(C, A), 3: jac.khatri_rao(B, A)}[mode]
    X, *_ = np.linalg.lstsq(KR, jac.unfold(t, mode).T, rcond=None)
    assert np.allclose(new[mode - 1], X.T, atol=1e-12)


def test_monotone_and_fixed_point():
    I, J, K, R = 8, 7, 6, 3
    T, _ = noisy(I, J, K, R, 0.1, 3)
    w0 = RNG.standard_normal(R * (I + J + K))
    f0, _ = oracle.cpd_eval(T, w0, I, J, K, R)
    _, fs = ALS.als(T, w0, I, J, K, R, 4)
    seq = np.concatenate([[f0], fs])
    assert np.all(np.diff(seq) <= 1e-12 * seq[:-1])
    # exact rank: the true factors are a fixed point of a sweep
    T0, (A, B, C) = noisy(I, J, K, R, 0.0, 4)
    w_true = ALS._pack([A, B, C])
    w1, fs1 = ALS.als(T0, w_true, I, J, K, R, 1)
    assert np.allclose(w1, w_true, atol=1e-10)
    assert np.all(fs1 <= 1e-20)


def test_mttkrp_matches_oracle_gradient_identity():
    """MTTKRP by the explicit unfolding equals W Π^(l) − ∂F/∂W^(l) (Kolda's gradient thm),
    with ∇F from the pinned oracle.cpd_eval."""
    I, J, K, R = 5, 4, 6, 3
    T, _ = noisy(I, J, K, R, 0.5, 7)
    w = RNG.standard_normal(R * (I + J + K))
    Ws = ALS._factors(w, I, J, K, R)
    _, g = oracle.cpd_eval(T, w, I, J, K, R)
    A, B, C = Ws
    P = [(B.T @ B) * (C.T @ C), (A.T @ A) * (C.T @ C), (A.T @ A) * (B.T @ B)]
    G = ALS._factors(g, I, J, K, R)
    for mode in (1, 2, 3):
        M = ALS.mttkrp(T, Ws, mode, I, J, K)
        assert np.allclose(M, Ws[mode - 1] @ P[mode - 1] - G[mode - 1], atol=1e-12)
