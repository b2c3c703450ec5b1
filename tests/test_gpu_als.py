"""Parity of the CUDA CP-ALS path (NEXT #4: single-mode MTTKRPs, Alg. ALS sweeps) with oracle/als.py.

Bars: an MTTKRP is a plain contraction — ‖ΔM‖ ≤ 1e-12·‖T‖‖⊙W‖-scale (we use 1e-12·‖M_ref‖ plus the
fp64 floor u·Σ|t||w||w| ≈ u·‖T‖·‖W‖‖W‖); an ALS update divides by V = Hadamard of Grams, so its error is
amplified by cond(V): compared within 1e-10·cond(V) relative (R30).
"""
import math

import numpy as np
import pytest
import torch

import oracle
import synth
from oracle import als as ALS
from oracle import jacobian as jac
from parity_util import TOL, to_np

pytestmark = pytest.mark.gpu
tf = pytest.importorskip("paper_2110_05997_b200")
U_ = 2.0 ** -53


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    c = tf.Context(0)
    yield c
    c.close()


def colmaj(flat, n, R):
    return np.asarray(flat, dtype=np.float64).reshape(R, n).T


def problem(I, J, K, R, seed, ldT=None):
    T = synth.randn((K, J, ldT or I), torch.device("cpu"), "als-test", seed, I, J, K)
    w = synth.randn((R * (I + J + K),), torch.device("cpu"), "als-w", seed, I, J, K, R)
    return T, w


@pytest.mark.parametrize("dims", [(6, 5, 4, 3), (37, 29, 23, 7), (130, 70, 90, 20), (200, 200, 200, 10),
                                  (64, 48, 40, 100), (50, 40, 30, 128)])
def test_mttkrp_modes(ctx, dims):
    I, J, K, R = dims
    T, w = problem(I, J, K, R, 1)
    Tn, wn = to_np(T).reshape(-1), to_np(w)
    Ws = ALS._factors(wn, I, J, K, R)
    d = tf.Dims(I, J, K, R)
    for mode, n in ((1, I), (2, J), (3, K)):
        M = colmaj(to_np(ctx.tf_mttkrp(d, T.cuda(), w.cuda(), mode)), n, R)
        ref = ALS.mttkrp(Tn, Ws, mode, I, J, K)
        scale = np.linalg.norm(Tn) * np.prod([np.linalg.norm(Ws[m]) for m in range(3) if m != mode - 1])
        assert np.linalg.norm(M - ref) <= 1e-12 * np.linalg.norm(ref) + 8 * U_ * scale, (mode, np.linalg.norm(M - ref))


def test_mttkrp_padded_and_sharded(ctx):
    """ldT = I + 3 (odd: the cp.async operand path) and a K-shard (modes 1, 2 partial sums; mode 3 local rows)."""
    I, J, K, R = 45, 33, 27, 6
    Tp, w = problem(I, J, K, R, 2, ldT=I + 3)
    wn = to_np(w)
    Tn = to_np(Tp[:, :, :I]).reshape(-1)
    Ws = ALS._factors(wn, I, J, K, R)
    for mode, n in ((1, I), (2, J), (3, K)):
        M = colmaj(to_np(ctx.tf_mttkrp(tf.Dims(I, J, K, R, ldT=I + 3), Tp.cuda(), w.cuda(), mode)), n, R)
        assert np.allclose(M, ALS.mttkrp(Tn, Ws, mode, I, J, K), rtol=0, atol=1e-11)
    k0, k1 = 10, 22
    Ts = Tp[k0:k1].contiguous()
    d = tf.Dims(I, J, k1 - k0, R, ldT=I + 3, K_total=K, k_begin=k0)
    t = jac.tensor_from_storage(Tn, I, J, K)
    sub = jac.storage_from_tensor(t[:, :, k0:k1])
    Wsub = [Ws[0], Ws[1], Ws[2][k0:k1]]
    for mode, n in ((1, I), (2, J), (3, k1 - k0)):
        M = colmaj(to_np(ctx.tf_mttkrp(d, Ts.cuda(), w.cuda(), mode)), n, R)
        assert np.allclose(M, ALS.mttkrp(sub, Wsub, mode, I, J, k1 - k0), rtol=0, atol=1e-11)


@pytest.mark.parametrize("dims,sweeps", [((20, 20, 20, 3), 1), ((37, 29, 23, 5), 3), ((120, 100, 80, 20), 2)])
def test_als_sweeps(ctx, dims, sweeps):
    I, J, K, R = dims
    A, B, C = (synth.randn((n, R), torch.device("cpu"), "als-true", n).numpy() for n in (I, J, K))
    t = np.einsum("ir,jr,kr->ijk", A, B, C) + 0.05 * synth.randn((I, J, K), torch.device("cpu"), "als-n").numpy()
    Tn = jac.storage_from_tensor(t)
    w0 = synth.randn((R * (I + J + K),), torch.device("cpu"), "als-w0", I).numpy()
    wref, fref = ALS.als(Tn, w0, I, J, K, R, sweeps)
    wt = torch.from_numpy(w0.copy()).cuda()
    fh = ctx.tf_als(tf.Dims(I, J, K, R), torch.from_numpy(Tn).cuda(), wt, sweeps, track_f=True)
    assert np.allclose(fh, fref, rtol=1e-9, atol=0), (fh, fref)
    assert np.linalg.norm(to_np(wt) - wref) <= 1e-8 * np.linalg.norm(wref)


def test_als_exact_rank_fixed_point(ctx):
    I, J, K, R = 30, 25, 20, 4
    A, B, C = (synth.randn((n, R), torch.device("cpu"), "als-fp", n).numpy() for n in (I, J, K))
    Tn = jac.storage_from_tensor(np.einsum("ir,jr,kr->ijk", A, B, C))
    w = ALS._pack([A, B, C])
    wt = torch.from_numpy(w.copy()).cuda()
    fh = ctx.tf_als(tf.Dims(I, J, K, R), torch.from_numpy(Tn).cuda(), wt, 1, track_f=True)
    assert np.all(fh <= 1e-20 * np.sum(Tn ** 2))
    assert np.allclose(to_np(wt), w, atol=1e-10 * np.abs(w).max())


@pytest.mark.slow
def test_c5_full_size_mttkrp_sampled(ctx):
    """c5 at full size in the bench's configuration: sampled rows of the three MTTKRPs against the oracle. A row of
    T_(1)(C ⊙ B) is the gradient row of the hyperslice S_i at a zero factor row (the residual is then S_i itself:
    -dF/dA[i] = sum_jk t_ijk B_j: C_k:, Lemma partialf), which oracle.slice_eval computes in 80-bit arithmetic."""
    import oracle
    Pb = synth.make_problem("c5", "cuda")
    c = Pb.cfg
    I, J, K, R = c.I, c.J, c.K, c.R
    w = Pb.w("random")
    d = tf.Dims(I, J, K, R)
    Ms = [ctx.tf_mttkrp(d, Pb.T, w, m).reshape(R, n).T.cpu().numpy() for m, n in ((1, I), (2, J), (3, K))]
    A, B, C = ALS._factors(to_np(w), I, J, K, R)
    zero = np.zeros(R)
    for i in (0, 517, I - 1):
        S = Pb.T[:, :, i].cpu().numpy().T            # S[j, k] = t[i, j, k]
        ref = -oracle.slice_eval(S, zero, B, C)[1]
        assert np.linalg.norm(Ms[0][i] - ref) <= TOL * np.linalg.norm(ref)
    for j in (0, 801, J - 1):
        S = Pb.T[:, j, :].cpu().numpy().T            # S[i, k]
        ref = -oracle.slice_eval(S, zero, A, C)[1]
        assert np.linalg.norm(Ms[1][j] - ref) <= TOL * np.linalg.norm(ref)
    for k in (0, 333, K - 1):
        S = Pb.T[k].cpu().numpy().T                   # S[i, j]
        ref = -oracle.slice_eval(S, zero, A, B)[1]
        assert np.linalg.norm(Ms[2][k] - ref) <= TOL * np.linalg.norm(ref)


def test_argument_errors_new_calls(ctx):
    """The compression / ALS / sharded-dGN calls return their documented status codes (no exceptions or exits
    across the ABI)."""
    T = torch.zeros(4 * 5 * 6, dtype=torch.float64, device="cuda")
    w = torch.zeros(3 * 15, dtype=torch.float64, device="cuda")
    with pytest.raises(tf.TfError) as ei:
        ctx.tf_mttkrp(tf.Dims(4, 5, 6, 3), T, w, 4)
    assert ei.value.status == tf.TF_ERR_ARG
    with pytest.raises(tf.TfError) as ei:   # compression needs the whole tensor
        ctx.tf_unfolding_grams(tf.Dims(4, 5, 3, 1, K_total=6, k_begin=3), T[:60].contiguous())
    assert ei.value.status == tf.TF_ERR_UNSUPPORTED
    with pytest.raises(tf.TfError) as ei:
        ctx.tf_sym_eig_top(4, torch.eye(4, dtype=torch.float64, device="cuda").reshape(-1), 5,
                           torch.zeros(20, dtype=torch.float64, device="cuda"))
    assert ei.value.status == tf.TF_ERR_ARG
    with pytest.raises(tf.TfError) as ei:   # tf_als on a shard
        ctx.tf_als(tf.Dims(4, 5, 3, 3, K_total=6, k_begin=0), T, w, 1)
    assert ei.value.status == tf.TF_ERR_UNSUPPORTED
    with pytest.raises(tf.TfError) as ei:   # energy init with more terms than core entries
        ctx.tf_energy_init(1, 1, 2, torch.ones(2, dtype=torch.float64, device="cuda"), 3)
    assert ei.value.status == tf.TF_ERR_ARG
    with pytest.raises(tf.TfError) as ei:
        ctx.set_eval_form("pi")
        ctx.tf_compress(tf.Dims(4, 5, 6, 3), T, torch.zeros(45, dtype=torch.float64, device="cuda"), mlsvd_tol=0.0)
    assert ei.value.status == tf.TF_ERR_ARG
    ctx.set_eval_form("auto")
    # a failing all-reduce hook surfaces as an exception, not a crash
    def bad(buf):
        raise RuntimeError("hook failed")
    with pytest.raises(RuntimeError):
        ctx.tf_cpd_dgn_sharded(tf.Dims(4, 5, 6, 3), T + 1.0, w + 0.5, [2] * 3, bad, maxiter=3)
