"""Parity of the CUDA compression stage (NEXT #3: unfolding Grams, truncated MLSVD by subspace iteration,
multilinear core, Alg. Compression, energy initialisation, uncompression) with oracle/mlsvd.py.

Bars: the unfolding Grams and the core are plain contractions — ‖Δ‖ ≤ 1e-12·‖ref‖ (fp64 sums of up to 10^6
products; the oracle rounds once per product in numpy/BLAS). The eigenpairs follow from them: eigenvalues
within 1e-10·λ_j + 64·sqrt(n)·u·λ_1 (the absolute fp64 floor of ANY eigensolver on the Gram), eigenvectors
(signs fixed by reading R23) within 1e-10 + 64·sqrt(n)·u·λ_1/gap_j — only where the gap makes them unique
(R23, R27).
"""
import json
import math
import os

import numpy as np
import pytest
import torch

import synth
from oracle import jacobian as jac
from oracle import mlsvd as M
from parity_util import to_np

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


def warmup_T(golden_dir):
    g = json.load(open(os.path.join(golden_dir, "warmup.json")))
    x, y = np.array(g["x"]), np.array(g["y"])
    z = np.array(g["z_num"], dtype=np.float64) / g["z_den"]
    X, Y, Z = np.meshgrid(x, y, z, indexing="ij")
    t = (np.cos(1 - X) * np.sin(1 + Y ** 2) - np.sin(1 + X ** 2) * np.exp(X ** 2 + Y ** 2 + Z ** 2)
         - np.cos(X) * np.log(1 + Z))
    return jac.storage_from_tensor(t)


def rand_T(I, J, K, seed, ldT=None):
    T = synth.randn((K, J, ldT or I), torch.device("cpu"), "mlsvd-test", seed, I, J, K)
    return T


def colmaj(flat, n, P):
    return np.asarray(flat, dtype=np.float64).reshape(P, n).T


def check_eig(lam, U, lam_ref, U_ref, n, tag="", base=1e-10):
    lam1 = abs(lam_ref[0])
    floor = 64 * math.sqrt(n) * U_ * lam1
    assert np.all(np.abs(lam - lam_ref) <= 1e-10 * np.abs(lam_ref) + floor), (tag, np.abs(lam - lam_ref).max())
    P = len(lam_ref)
    for j in range(P):
        gaps = [abs(lam_ref[j] - lam_ref[i]) for i in range(P) if i != j]
        gap = min(gaps) if gaps else lam1
        if gap <= 1e-6 * lam1:
            continue   # eigenvector not unique to the precision of the data
        err = np.linalg.norm(U[:, j] - U_ref[:, j])
        assert err <= base + 64 * math.sqrt(n) * U_ * lam1 / gap, (tag, j, err, gap / lam1)


# ------------------------------------------------------------------------- unfolding Grams
@pytest.mark.parametrize("dims", [(6, 5, 4), (37, 29, 23), (130, 70, 90), (200, 200, 200)])
def test_unfolding_grams(ctx, dims):
    I, J, K = dims
    T = rand_T(I, J, K, 1)
    Tn = to_np(T).reshape(-1)
    Gs = ctx.tf_unfolding_grams(tf.Dims(I, J, K, 1), T.cuda())
    torch.cuda.synchronize()
    for mode, n in ((1, I), (2, J), (3, K)):
        G = to_np(Gs[mode - 1]).reshape(n, n).T
        ref = M.unfolding_gram(Tn, I, J, K, mode)
        assert np.linalg.norm(G - ref) <= 1e-12 * np.linalg.norm(ref), (mode, np.linalg.norm(G - ref))
        assert np.array_equal(G, G.T)


def test_unfolding_grams_padded_ld(ctx):
    """T with a padded leading dimension ldT = I + 3 (odd: the cp.async operand path) and ldT = I + 2."""
    I, J, K = 45, 33, 27
    for ldT in (I + 3, I + 2):
        Tp = rand_T(I, J, K, 2, ldT=ldT)
        Tn = to_np(Tp[:, :, :I]).reshape(-1)
        Gs = ctx.tf_unfolding_grams(tf.Dims(I, J, K, 1, ldT=ldT), Tp.cuda())
        torch.cuda.synchronize()
        for mode, n in ((1, I), (2, J), (3, K)):
            G = to_np(Gs[mode - 1]).reshape(n, n).T
            ref = M.unfolding_gram(Tn, I, J, K, mode)
            assert np.linalg.norm(G - ref) <= 1e-12 * np.linalg.norm(ref), (ldT, mode)


# ------------------------------------------------------------------------- eigenpairs
@pytest.mark.parametrize("n,P", [(6, 3), (29, 7), (200, 10), (301, 64), (257, 128)])
def test_sym_eig_top(ctx, n, P):
    rng = np.random.default_rng(n * 1000 + P)
    X = rng.standard_normal((n, n + 40))
    X[:, :P] *= np.linspace(40, 5, P)   # a spectrum with a gap after P
    G = X @ X.T
    U_ref, _, lam_ref = M.mode_svd(G, P)
    Om = synth.randn((P, n), torch.device("cpu"), "eig-test", n, P).reshape(-1)
    Ud, lam, it = ctx.tf_sym_eig_top(n, torch.from_numpy(G.T.copy().reshape(-1)).cuda(), P, Om.cuda())
    torch.cuda.synchronize()
    check_eig(to_np(lam), colmaj(to_np(Ud), n, P), lam_ref, U_ref, n, (n, P))
    Uh = colmaj(to_np(Ud), n, P)
    assert np.abs(Uh.T @ Uh - np.eye(P)).max() < 1e-13
    assert 1 <= it <= 100


def test_sym_eig_rank_deficient(ctx):
    """G of rank 3 with P = 6: three ~0 eigenvalues (their vectors are not unique) — the leading three
    match and the block stays orthonormal (Householder handles the null directions)."""
    n, P = 40, 6
    rng = np.random.default_rng(5)
    X = rng.standard_normal((n, 3))
    G = X @ X.T
    U_ref, _, lam_ref = M.mode_svd(G, P)
    Om = synth.randn((P, n), torch.device("cpu"), "eig-rd").reshape(-1)
    Ud, lam, it = ctx.tf_sym_eig_top(n, torch.from_numpy(G.T.copy().reshape(-1)).cuda(), P, Om.cuda())
    torch.cuda.synchronize()
    lam = to_np(lam)
    Uh = colmaj(to_np(Ud), n, P)
    assert np.abs(lam[3:]).max() <= 64 * math.sqrt(n) * U_ * lam_ref[0]
    check_eig(lam[:3], Uh[:, :3], lam_ref[:3], U_ref[:, :3], n)
    assert np.abs(Uh.T @ Uh - np.eye(P)).max() < 1e-13


# ------------------------------------------------------------------------- core and the whole compression
@pytest.mark.parametrize("dims,P", [((6, 5, 4), (3, 3, 3)), ((37, 29, 23), (7, 5, 9)), ((130, 70, 90), (20, 13, 40)),
                                    ((64, 200, 66), (64, 100, 2))])
def test_multilinear_core(ctx, dims, P):
    I, J, K = dims
    T = rand_T(I, J, K, 3)
    Tn = to_np(T).reshape(-1)
    rng = np.random.default_rng(sum(dims))
    Us = [np.linalg.qr(rng.standard_normal((n, p)))[0] for n, p in zip(dims, P)]
    S = ctx.tf_multilinear_core(tf.Dims(I, J, K, 1), T.cuda(),
                                *[x for U, p in zip(Us, P) for x in (torch.from_numpy(U.T.copy().reshape(-1)).cuda(), p)])
    torch.cuda.synchronize()
    ref = M.multilinear(Tn, I, J, K, Us[0].T, Us[1].T, Us[2].T)
    got = to_np(S).reshape(P[2], P[1], P[0]).transpose(2, 1, 0)
    assert np.linalg.norm(got - ref) <= 1e-12 * np.linalg.norm(Tn), np.linalg.norm(got - ref)


def _compress(ctx, Tn_t, I, J, K, R, tol):
    Om = synth.omega_blocks((I, J, K), R, "cpu")
    out = ctx.tf_compress(tf.Dims(I, J, K, R), Tn_t.cuda(), Om.cuda(), mlsvd_tol=tol)
    torch.cuda.synchronize()
    return out


def test_compress_warmup_table_4_5(ctx, golden_dir):
    """Alg. Compression on the warming-up tensor through the CUDA path: ranks (3, 3, 3), and the GPU core
    reproduces Table 4.5 to its 8 printed decimals and the printed core magnitudes."""
    T = warmup_T(golden_dir)
    g = json.load(open(os.path.join(golden_dir, "warmup_mlsvd.json")))
    out = _compress(ctx, torch.from_numpy(T), 6, 5, 4, 3, 1e-6)
    assert out["ranks"] == (3, 3, 3)
    S = to_np(out["S"]).reshape(3, 3, 3).transpose(2, 1, 0)
    for shape, printed in g["table_4_5"]:
        assert abs(M.truncation_error(S, shape) - printed) <= 0.5e-8 + 1e-12, shape
    ref = M.compress(T, 6, 5, 4, 3, 1e-6)
    assert np.linalg.norm(S - ref["S"]) <= 1e-12 * np.linalg.norm(T)
    for l, n in enumerate((6, 5, 4)):
        assert np.allclose(to_np(out["sigma"][l]), ref["sigma"][l], rtol=1e-12, atol=1e-12 * ref["sigma"][l][0])
    # energy initialisation on the GPU core: the paper's picks and 0.0153 initial error
    w = to_np(ctx.tf_energy_init(3, 3, 3, out["S"].contiguous(), 3))
    W1, W2, W3, _ = M.energy_init(ref["S"], 3)
    assert np.allclose(w, np.concatenate([W1.T.reshape(-1), W2.T.reshape(-1), W3.T.reshape(-1)]), atol=1e-12)
    Ws = [torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in (W1.T.reshape(-1), W2.T.reshape(-1),
                                                                       W3.T.reshape(-1))]
    fac = [colmaj(to_np(ctx.tf_uncompress(n, 3, out["U"][l].contiguous(), Ws[l], 3)), n, 3)
           for l, n in enumerate((6, 5, 4))]
    t = jac.tensor_from_storage(T, 6, 5, 4)
    rec = np.einsum("ir,jr,kr->ijk", *fac)
    err = np.linalg.norm(t - rec) / np.linalg.norm(t)
    assert 0.0153 <= err < 0.0154, err


@pytest.mark.parametrize("name,dims,tol", [("c1", None, 1e-6), ("c2", None, 1e-6), ("c3", (120, 100, 80, 20), 1e-4),
                                           ("c4", (200, 96, 50, 30), 1e-6), ("c5", (100, 77, 21, 100), 1e-6)])
def test_compress_recipes(ctx, name, dims, tol):
    """The whole compression on the seeded recipes (reduced where the oracle needs it): ranks equal, sigma,
    U (where unique) and the truncated core match the oracle."""
    Pb = synth.make_problem(name, "cpu", dims=dims)
    c = Pb.cfg
    I, J, K, R = c.I, c.J, c.K, c.R
    Tn = to_np(Pb.T).reshape(-1)
    out = _compress(ctx, Pb.T, I, J, K, R, tol)
    ref = M.compress(Tn, I, J, K, R, tol)
    assert out["ranks"] == ref["ranks"], (out["ranks"], ref["ranks"])
    for l, n in enumerate((I, J, K)):
        P = min(n, R)
        lam_ref = ref["full"]["lam"][l]
        check_eig(to_np(out["sigma"][l]) ** 2, colmaj(to_np(out["U"][l]), n, P), lam_ref, ref["full"]["U"][l], n,
                  (name, l))
    r1, r2, r3 = ref["ranks"]
    S = to_np(out["S"]).reshape(r3, r2, r1).transpose(2, 1, 0)
    # the core inherits the eigenvector accuracy: compare where every mode's vectors are unique
    err = np.linalg.norm(S - ref["S"]) / np.linalg.norm(Tn)
    assert err <= 1e-9, err


def test_compress_exact_rank_recovers_factors(ctx):
    """Remark mlsvd-cpd: for T = [[A,B,C]] the compressed core is [[U1^T A, U2^T B, U3^T C]]
    — the GPU core, contracted back with the GPU U's, reproduces T to fp64 accuracy."""
    I, J, K, R = 50, 40, 30, 4
    A, B, C = (synth.randn((n, R), torch.device("cpu"), "exact", n).numpy() for n in (I, J, K))
    t = np.einsum("ir,jr,kr->ijk", A, B, C)
    T = jac.storage_from_tensor(t)
    out = _compress(ctx, torch.from_numpy(T), I, J, K, R, 1e-10)
    assert out["ranks"] == (4, 4, 4)
    Us = [colmaj(to_np(out["U"][l]), n, 4) for l, n in enumerate((I, J, K))]
    S = to_np(out["S"]).reshape(4, 4, 4).transpose(2, 1, 0)
    rec = np.einsum("ia,jb,kc,abc->ijk", *Us, S)
    assert np.linalg.norm(rec - t) <= 1e-12 * np.linalg.norm(t)


@pytest.mark.slow
def test_c5_full_size_compression_sampled(ctx):
    """c5 (1200³, R=100) through the CUDA compression in the bench's launch configuration: orthonormal U,
    sigma² sums within ‖T‖², sampled Gram entries (hyperslice inner products) and sampled
    core entries s_abc = Σ_k U3[k,c] u1_a^T T_k u2_b recomputed on the host."""
    Pb = synth.make_problem("c5", "cuda")
    c = Pb.cfg
    I, J, K, R = c.I, c.J, c.K, c.R
    d = tf.Dims(I, J, K, R)
    Gs = ctx.tf_unfolding_grams(d, Pb.T, modes=(1,))
    G1 = Gs[0].reshape(I, I).T
    Th = Pb.T.cpu().numpy().reshape(-1)
    rng = np.random.default_rng(11)
    for p, q in [(0, 0), (I - 1, 3)] + [tuple(rng.choice(I, 2)) for _ in range(2)]:
        ref = M.gram_entry(Th, I, J, K, 1, int(p), int(q))
        assert abs(G1[p, q].item() - ref) <= 1e-12 * math.sqrt(G1[p, p].item() * G1[q, q].item())
    del Gs, G1
    Om = synth.omega_blocks((I, J, K), R, "cuda")
    out = ctx.tf_compress(d, Pb.T, Om, mlsvd_tol=1e-6)
    torch.cuda.synchronize()
    assert out["ranks"] == (100, 100, 100)
    nT2 = float(torch.sum(Pb.T * Pb.T))
    for l, n in enumerate((I, J, K)):
        Ul = out["U"][l].reshape(100, n)
        assert (Ul @ Ul.T - torch.eye(100, device=Ul.device, dtype=torch.float64)).abs().max().item() < 1e-13
        s2 = float(torch.sum(out["sigma"][l] ** 2))
        assert s2 <= nT2 * (1 + 1e-12) and s2 >= 0.99 * nT2
    S = out["S"].reshape(100, 100, 100)          # S[c, b, a]
    U1 = out["U"][0].reshape(100, I).cpu().numpy()
    U2 = out["U"][1].reshape(100, J).cpu().numpy()
    U3 = out["U"][2].reshape(100, K).cpu().numpy()
    T3 = Th.reshape(K, J, I)
    for a, b, cc in [(0, 0, 0), (99, 50, 7)]:
        acc = 0.0
        for k in range(K):
            acc += U3[cc, k] * float(U2[b] @ (T3[k] @ U1[a]))
        assert abs(S[cc, b, a].item() - acc) <= 1e-11 * math.sqrt(nT2), (a, b, cc)


# ------------------------------------------------------------------------- the whole Tensor Fox flow
def _oracle_pipeline(T, I, J, K, R, tol, cgi, maxiter, w0_blocks=None, dgn_tol=1e-6):
    import oracle
    c = M.compress(T, I, J, K, R, tol)
    r1, r2, r3 = c["ranks"]
    if w0_blocks is None:
        W1, W2, W3, _ = M.energy_init(c["S"], R)
    else:
        W1, W2, W3 = (blk[:r] for blk, r in zip(w0_blocks, c["ranks"]))
    w0 = np.concatenate([W1.T.reshape(-1), W2.T.reshape(-1), W3.T.reshape(-1)])
    Sflat = jac.storage_from_tensor(c["S"])
    ref = oracle.dgn(Sflat, w0, r1, r2, r3, R, cgi, maxiter=maxiter, tol=dgn_tol)
    w = ref["w"]
    Ws = [w[:R * r1].reshape(R, r1).T, w[R * r1:R * (r1 + r2)].reshape(R, r2).T, w[R * (r1 + r2):].reshape(R, r3).T]
    full = M.uncompress(c["U"], Ws)
    unit, lam = M.normalize_cpd(full)
    return c, ref, unit, lam


def test_tf_cpd_warmup(ctx, golden_dir):
    """Compression -> energy initialisation -> dGN -> uncompression on the warming-up tensor:
    the GPU flow follows the oracle's flow (same ranks, same first dGN iterates) and, with tol = 1e-12, fits T to
    the order of the paper's printed final CPD (relative error 5.6e-7): below 1e-6. Long dGN runs
    are chaotic in the last bits (different fp64 summation orders), so only the first iterations are compared
    entry by entry and the end point by its quality."""
    T = warmup_T(golden_dir)
    cgi = synth.cg_budget(200, seed=9)
    Om = synth.omega_blocks((6, 5, 4), 3, "cpu")
    W, lam, out, hist = ctx.tf_cpd(tf.Dims(6, 5, 4, 3), torch.from_numpy(T).cuda(), Om.cuda(), cgi, tol=1e-12)
    c, ref, unit, lam_ref = _oracle_pipeline(T, 6, 5, 4, 3, 1e-6, cgi, None, dgn_tol=1e-12)
    assert out["ranks"] == c["ranks"] == (3, 3, 3)
    n0 = min(10, len(hist), len(ref["hist"]))
    assert np.allclose(hist[:n0, 0], ref["hist"][:n0, 0], rtol=1e-8, atol=0)
    assert np.array_equal(hist[:n0, 2], ref["hist"][:n0, 2]) or np.allclose(hist[:n0, 2], ref["hist"][:n0, 2],
                                                                           rtol=1e-12)
    assert out["rel_err"] < 1e-6 and ref["hist"][-1, 1] < 1e-6, (out, ref["hist"][-1])
    Wn = to_np(W)
    t = jac.tensor_from_storage(T, 6, 5, 4)
    a, b, cc = (Wn[:18].reshape(3, 6).T, Wn[18:33].reshape(3, 5).T, Wn[33:].reshape(3, 4).T)
    for X in (a, b, cc):
        assert np.allclose(np.linalg.norm(X, axis=0), 1.0, atol=1e-14)
    rec = np.einsum("r,ir,jr,kr->ijk", to_np(lam), a, b, cc)
    assert abs(np.linalg.norm(t - rec) / np.linalg.norm(t) - out["rel_err"]) <= 1e-2 * out["rel_err"] + 1e-14


def test_tf_cpd_random_init_recipe(ctx):
    """The flow with a random N(0,1) start on the core on a reduced c3 recipe (collinear
    factors, noise), a fixed number of dGN iterations: the trajectory and the uncompressed factors match the
    oracle's flow."""
    Pb = synth.make_problem("c3", "cpu", dims=(60, 50, 40, 5))
    c = Pb.cfg
    I, J, K, R = c.I, c.J, c.K, c.R
    T = to_np(Pb.T).reshape(-1)
    cgi = synth.cg_budget(12, seed=2)
    Ps = [min(n, R) for n in (I, J, K)]
    blocks = [synth.randn((R, p), torch.device("cpu"), "core-init", l).numpy().T for l, p in enumerate(Ps)]
    w0 = torch.from_numpy(np.concatenate([b.T.reshape(-1) for b in blocks]))
    Om = synth.omega_blocks((I, J, K), R, "cpu")
    W, lam, out, hist = ctx.tf_cpd(tf.Dims(I, J, K, R), Pb.T.cuda(), Om.cuda(), cgi, w0_core=w0.cuda(), maxiter=12,
                                   tol=0.0)
    cref, ref, unit, lam_ref = _oracle_pipeline(T, I, J, K, R, 1e-6, cgi, 12, w0_blocks=blocks, dgn_tol=0.0)
    assert out["ranks"] == cref["ranks"]
    assert out["dgn"]["iters"] == ref["iters"] == 12
    assert np.allclose(hist[:, 0], ref["hist"][:, 0], rtol=1e-7)
    assert np.allclose(hist[:, 2], ref["hist"][:, 2], rtol=1e-12)
    Wr = np.concatenate([u.T.reshape(-1) for u in unit])
    assert np.linalg.norm(to_np(W) - Wr) <= 1e-6 * np.linalg.norm(Wr)
    assert np.allclose(to_np(lam), lam_ref, rtol=1e-6)


@pytest.mark.parametrize("name,dims,tol", [("c1", None, 1e-6), ("c2", None, 1e-6), ("c3", (120, 100, 80, 20), 1e-4),
                                           ("c4", (200, 96, 50, 30), 1e-6), ("warmup", None, 1e-6)])
def test_compress_st_matches_oracle(ctx, name, dims, tol, golden_dir):
    """Alg. ST-MLSVD through the CUDA path (tf_compress_st) against oracle st_mlsvd: ranks, each step's sigma and
    U (where unique), and the core. Steps 2 and 3 work on the intermediate X1 = U~1^T T_(1) (and X2), so the
    step-1 eigenvector error (~1e-11 where gaps are small, e.g. the warming-up tensor's sigma_3 = 0.13 against
    sigma_1 = 45.9) is carried into their Grams: their eigenvector bar is 1e-9 instead of 1e-10."""
    if name == "warmup":
        T = warmup_T(golden_dir)
        I, J, K, R = 6, 5, 4, 3
        Tt = torch.from_numpy(T)
    else:
        Pb = synth.make_problem(name, "cpu", dims=dims)
        c = Pb.cfg
        I, J, K, R = c.I, c.J, c.K, c.R
        T = to_np(Pb.T).reshape(-1)
        Tt = Pb.T
    Om = synth.omega_blocks((I, J, K), R, "cpu")
    out = ctx.tf_compress(tf.Dims(I, J, K, R), Tt.cuda(), Om.cuda(), mlsvd_tol=tol, sequential=True)
    torch.cuda.synchronize()
    ref = M.st_mlsvd(T, I, J, K, R, tol)
    assert out["ranks"] == ref["ranks"]
    rs = [I, ref["ranks"][0], ref["ranks"][0]]
    for l, n in enumerate((I, J, K)):
        P = min(n, R)
        lam_ref = ref["sigma"][l] ** 2
        check_eig(to_np(out["sigma"][l]) ** 2, colmaj(to_np(out["U"][l]), n, P), lam_ref, ref["Ufull"][l], n,
                  (name, l), base=1e-10 if l == 0 else 1e-9)
    r1, r2, r3 = ref["ranks"]
    S = to_np(out["S"]).reshape(r3, r2, r1).transpose(2, 1, 0)
    assert np.linalg.norm(S - ref["S"]) / np.linalg.norm(T) <= 1e-9


def test_tf_cpd_sequential_compression(ctx):
    """The flow with ST-MLSVD compression on an exact-rank tensor (no truncation loss): converges to a fit below
    1e-6 and the unit-column output reproduces T to that fit."""
    I, J, K, R = 40, 30, 20, 3
    A, B, C = (synth.randn((n, R), torch.device("cpu"), "cpd-st", n).numpy() for n in (I, J, K))
    t = np.einsum("ir,jr,kr->ijk", A, B, C)
    T = jac.storage_from_tensor(t)
    cgi = synth.cg_budget(200, seed=3)
    Om = synth.omega_blocks((I, J, K), R, "cpu")
    W, lam, out, hist = ctx.tf_cpd(tf.Dims(I, J, K, R), torch.from_numpy(T).cuda(), Om.cuda(), cgi, tol=1e-12,
                                   sequential=True)
    assert out["ranks"] == (3, 3, 3)
    assert out["rel_err"] < 1e-6, out
    Wn = to_np(W)
    a, b, c = (Wn[:I * R].reshape(R, I).T, Wn[I * R:(I + J) * R].reshape(R, J).T, Wn[(I + J) * R:].reshape(R, K).T)
    rec = np.einsum("r,ir,jr,kr->ijk", to_np(lam), a, b, c)
    assert abs(np.linalg.norm(t - rec) / np.linalg.norm(t) - out["rel_err"]) <= 1e-2 * out["rel_err"] + 1e-14


# ------------------------------------------------------------------------- K-sharded compression and flow
def _run_ranks(world, fn):
    """Run fn(rank, hook) on `world` host threads, each with its own context and stream on this GPU; hook(buf)
    sums the ranks' buffers on the host side (no kernel waits on another rank's kernels)."""
    import threading
    bufs = [None] * world
    outs = [None] * world
    errs = []
    barrier = threading.Barrier(world)

    def hook_for(rank):
        def hook(buf):
            bufs[rank] = buf
            barrier.wait()
            if rank == 0:
                total = bufs[0].clone()
                for r in range(1, world):
                    total += bufs[r]
                torch.cuda.synchronize()
                for r in range(world):
                    bufs[r].copy_(total)
                torch.cuda.synchronize()
            barrier.wait()
        return hook

    def run(rank):
        try:
            torch.cuda.set_device(0)
            stream = torch.cuda.Stream()
            with torch.cuda.stream(stream):
                c = tf.Context(0, stream)
                outs[rank] = fn(rank, c, hook_for(rank))
                torch.cuda.synchronize()
                c.close()
        except Exception as e:   # surface in the main thread
            errs.append(e)
            barrier.abort()

    ths = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    if errs:
        raise errs[0]
    return outs


@pytest.mark.parametrize("name,dims,world", [("c3", (80, 70, 60, 12), 3), ("c4", (120, 64, 40, 20), 2)])
def test_compress_st_sharded_matches_single_device(ctx, name, dims, world):
    """tf_compress_st_sharded over K-shards equals tf_compress_st on the whole tensor (only the reduction order of
    the all-reduced Grams differs): same ranks, sigma, U (where unique) and core; every rank holds the same."""
    from paper_2110_05997_b200.dist import shard_range
    Pb = synth.make_problem(name, "cpu", dims=dims)
    c = Pb.cfg
    I, J, K, R = c.I, c.J, c.K, c.R
    Om = synth.omega_blocks((I, J, K), R, "cpu").cuda()
    ref = ctx.tf_compress(tf.Dims(I, J, K, R), Pb.T.cuda(), Om, mlsvd_tol=1e-6, sequential=True)
    torch.cuda.synchronize()

    def fn(rank, c_, hook):
        k0, k1 = shard_range(K, rank, world)
        Tl = Pb.T[k0:k1].contiguous().cuda()
        out = c_.tf_compress_st_sharded(tf.Dims(I, J, k1 - k0, R, K_total=K, k_begin=k0), Tl, Om, hook,
                                        mlsvd_tol=1e-6)
        return {k: ([to_np(x) for x in v] if isinstance(v, list) and v and isinstance(v[0], torch.Tensor)
                    else (to_np(v) if isinstance(v, torch.Tensor) else v)) for k, v in out.items()}

    outs = _run_ranks(world, fn)
    for o in outs:
        assert o["ranks"] == ref["ranks"]
        for l, n in enumerate((I, J, K)):
            P = min(n, R)
            lam_ref = to_np(ref["sigma"][l]) ** 2
            check_eig(o["sigma"][l] ** 2, colmaj(o["U"][l], n, P), lam_ref, colmaj(to_np(ref["U"][l]), n, P), n,
                      (name, l), base=1e-9)
        assert np.linalg.norm(o["S"] - to_np(ref["S"])) <= 1e-9 * np.linalg.norm(to_np(Pb.T))
    for o in outs[1:]:
        assert np.array_equal(o["S"], outs[0]["S"])


def test_cpd_sharded_matches_single_device(ctx):
    """The K-sharded flow (tf_cpd_sharded) on 2 ranks against tf_cpd (sequential) on the whole tensor: same ranks,
    the dGN on the (identical up to rounding) core takes the same first steps, and the fits agree."""
    from paper_2110_05997_b200.dist import shard_range
    I, J, K, R = 40, 30, 24, 3
    A, B, C = (synth.randn((n, R), torch.device("cpu"), "cpd-shard", n).numpy() for n in (I, J, K))
    t = np.einsum("ir,jr,kr->ijk", A, B, C) + 1e-3 * synth.randn((I, J, K), torch.device("cpu"), "cpd-shard-n").numpy()
    T = torch.from_numpy(jac.storage_from_tensor(t)).reshape(K, J, I)
    Om = synth.omega_blocks((I, J, K), R, "cpu").cuda()
    cgi = synth.cg_budget(40, seed=8)
    W, lam, ref, href = ctx.tf_cpd(tf.Dims(I, J, K, R), T.reshape(-1).cuda(), Om, cgi, maxiter=40, tol=1e-10,
                                   sequential=True)
    world = 2

    def fn(rank, c_, hook):
        k0, k1 = shard_range(K, rank, world)
        Tl = T[k0:k1].contiguous().cuda()
        Wr, lr, out, hist = c_.tf_cpd_sharded(tf.Dims(I, J, k1 - k0, R, K_total=K, k_begin=k0), Tl, Om, cgi, hook,
                                              maxiter=40, tol=1e-10)
        return to_np(Wr), to_np(lr), out, hist

    outs = _run_ranks(world, fn)
    for Wr, lr, out, hist in outs:
        assert out["ranks"] == ref["ranks"]
        n0 = min(6, len(hist), len(href))
        assert np.allclose(hist[:n0, 0], href[:n0, 0], rtol=1e-8)
        assert abs(out["rel_err"] - ref["rel_err"]) <= 1e-3 * ref["rel_err"] + 1e-12
    assert np.array_equal(outs[0][0], outs[1][0])
