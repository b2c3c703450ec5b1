"""Parity at the full sizes the bench times (BASELINE.json configs c3 and c5), element by element.

* F and the WHOLE gradient vector of tf_cpd_eval against the oracle (not sampled rows): c3 at both points in
  both algebraic forms (reading R31), c5 in both forms. The oracle sums the definition slab by slab over k
  (F and dF/dA, dF/dB are sums over frontal slices, dF/dC row k depends on slice k only: PAPER.md:1844-1851,
  1801-1805), which is exactly the definition's sum split in k.
* Alg. CG-dGN in the launch configuration the bench times: c3 (n = 30 000, 10 iterations,
  lambda = 1e-3, Jacobi on/off, the collinear true point and a random point; once more on a 37-block grid) and c5
  (n = 360 000, 20 iterations, the row-owned persistent kernel on the full grid). Per iteration i: the GPU's x^(i)
  against
  the oracle's (iterate drift, reported), ||r^(i)||^2, and the GN matvec (Thm Hv) of the
  search direction the oracle's CG formed at that iteration, at 1e-10 per block and per element (per element the
  floor is the fp64 forward-error bound of the matvec's terms where the result cancels: parity_util.hv_abs_terms).
* The cancellation guard of the Pi form (reading R31) just above its thresholds: 2F/||T||^2 in {1.05e-3, 2e-3,
  1e-2} and ||grad F||/||W Pi|| = 1.1e-3, forced Pi form, against the oracle at 1e-10.
* Bitwise determinism of both forms at c3 full size.
* The K-sharded evaluation at c5 (2 and 8 shards): the shards' partial [grad | F] summed in rank order (the
  all-reduce) against the single-device result (1e-12) and the oracle (1e-10 per block and element).

Set TF_PARITY_REPORT=<dir> to write the per-iteration drift curves and error ratios as JSON.
"""
import json
import math
import os

import numpy as np
import pytest
import torch

import oracle
import synth
from parity_util import (TOL, U, block_floors, check_elementwise, check_elementwise_floor, f_floor, grad_floor,
                         hv_abs_terms, rel_err, to_np, w_blocks, within)

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

tf = pytest.importorskip("paper_2110_05997_b200")

_REPORT = {}


def _report(key, value):
    _REPORT[key] = value
    d = os.environ.get("TF_PARITY_REPORT")
    if d:
        os.makedirs(d, exist_ok=True)
        with open(os.path.join(d, "fullsize_parity.json"), "w") as fh:
            json.dump(_REPORT, fh, indent=1, default=float)


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    c = tf.Context(0)
    yield c
    c.close()


def oracle_eval_slabs(T_dev, w, I, J, K, R, slab=100):
    """The oracle's F and grad of the (K, J, I) device tensor T, slab by slab over k: F and dF/dA, dF/dB are
    sums over slices, row k of dF/dC depends on slice k only (the definition's sums split in k)."""
    w = to_np(w)
    A, B = w[:I * R], w[I * R:(I + J) * R]
    C_t = w[(I + J) * R:].reshape(R, K)
    f_parts = []
    gA, gB = np.zeros(I * R), np.zeros(J * R)
    gC_t = np.zeros((R, K))
    for k0 in range(0, K, slab):
        k1 = min(K, k0 + slab)
        Ts = T_dev[k0:k1].cpu().numpy().reshape(-1)
        ws = np.concatenate([A, B, np.ascontiguousarray(C_t[:, k0:k1]).reshape(-1)])
        fs, gs = oracle.cpd_eval(Ts, ws, I, J, k1 - k0, R)
        f_parts.append(fs)
        gA += gs[:I * R]
        gB += gs[I * R:(I + J) * R]
        gC_t[:, k0:k1] = gs[(I + J) * R:].reshape(R, k1 - k0)
    return math.fsum(f_parts), np.concatenate([gA, gB, gC_t.reshape(-1)])


def t_norm2(T_dev):
    return float(sum(float(torch.sum(T_dev[k0:k0 + 64] ** 2)) for k0 in range(0, T_dev.shape[0], 64)))


def check_eval_full(ctx, P, w, fr, gr, form, expect_fallback=None, T_np=None, key=""):
    c = P.cfg
    I, J, K, R = c.I, c.J, c.K, c.R
    ctx.set_eval_form(form)
    try:
        f, g = ctx.tf_cpd_eval(tf.Dims(I, J, K, R), P.T, w)
        torch.cuda.synchronize()
        fb = ctx.eval_fell_back()
    finally:
        ctx.set_eval_form("auto")
    if expect_fallback is not None:
        assert fb == expect_fallback, (key, form, fb)
    wn = to_np(w)
    nT2 = t_norm2(P.T)
    fl_f = 2.0 ** -53 * math.sqrt(nT2) * math.sqrt(2 * max(fr, 0.0)) + (2.0 ** -53) ** 2 * nT2
    okf, ef, bf = within([f.item()], [fr], fl_f)
    assert okf, (key, form, "f", ef, bf)
    g = to_np(g)
    okg, eg, bg = within(g, gr, grad_floor(wn, I, J, K, R))
    assert okg, (key, form, "grad", eg, bg)
    per = check_elementwise(g, gr, w_blocks(I, J, K, R), block_floors(wn, I, J, K, R))
    _report(f"eval/{key}/{form}", {"f_rel": ef / max(abs(fr), 1e-300), "grad_rel": eg / max(np.linalg.norm(gr), 1e-300),
                                   "fell_back": fb, "blocks": per})
    return g


# ------------------------------------------------------------------------------------------------ c3
@pytest.fixture(scope="module")
def c3():
    P = synth.make_problem("c3", "cuda")
    c = P.cfg
    ref = {}
    for point in ("true", "random"):
        ref[point] = oracle_eval_slabs(P.T, P.w(point), c.I, c.J, c.K, c.R)
    return P, ref


@pytest.mark.parametrize("point", ["true", "random"])
def test_c3_full_vector_eval(ctx, c3, point):
    """c3 (500^3, R = 20) full size: F and all 30 000 gradient entries, guarded Pi form (default at this size;
    at the collinear true point 2F/||T||^2 = 0.999e-3 < 1e-3, so the guard reruns the residual form) and the
    residual form, against the oracle per block and per element."""
    P, ref = c3
    fr, gr = ref[point]
    check_eval_full(ctx, P, P.w(point), fr, gr, "auto", expect_fallback=1 if point == "true" else 0, key=f"c3/{point}")
    check_eval_full(ctx, P, P.w(point), fr, gr, "residual", key=f"c3/{point}")


def test_c3_deterministic_bitwise(ctx, c3):
    """Reruns give bitwise-identical F and grad in both forms (fixed-order reductions), at the size the bench
    times (the Pi-form pass with its guard and, at the true point, the fallback)."""
    P, _ = c3
    c = P.cfg
    d = tf.Dims(c.I, c.J, c.K, c.R)
    for form, point in (("pi", "random"), ("pi", "true"), ("residual", "random")):
        ctx.set_eval_form(form)
        try:
            f1, g1 = ctx.tf_cpd_eval(d, P.T, P.w(point))
            f1, g1 = f1.clone(), g1.clone()
            for _ in range(2):
                f2, g2 = ctx.tf_cpd_eval(d, P.T, P.w(point))
                assert torch.equal(f1, f2) and torch.equal(g1, g2), (form, point)
        finally:
            ctx.set_eval_form("auto")


def _cg_parity(ctx, key, w, rhs, lam, iters, jacobi, I, J, K, R, x_bar):
    """Per-iteration CG parity; returns the drift curve. x_bar bounds the iterate drift (see the callers)."""
    ref = oracle.cg(w, rhs, lam, iters, I, J, K, R, jacobi=jacobi, history=True)
    assert ref["iters"] == iters and ref["status"] == 0
    d = tf.Dims(I, J, K, R)
    wt = torch.from_numpy(np.ascontiguousarray(w)).cuda()
    grams = ctx.tf_grams(d, wt)
    rt = torch.from_numpy(np.ascontiguousarray(rhs)).cuda()
    blocks = w_blocks(I, J, K, R)
    drift, r2err, mv = [], [], []
    x_prev = np.zeros_like(w)
    for i in range(1, iters + 1):
        x, it, r2 = ctx.tf_cg_solve(d, grams, wt, rt, lam, i, 0.0, jacobi)
        assert it == i
        xr = ref["x_hist"][i - 1]
        drift.append(rel_err(to_np(x), xr))
        r2err.append(abs(r2 - ref["r2"][i - 1]) / ref["r2"][0])
        # the GN matvec of the direction the oracle's CG formed at iteration i (w-coordinates:
        # x^(i) - x^(i-1) = alpha_i M^{-1/2} p_hat_i)
        v = (xr - x_prev) / ref["alpha"][i - 1]
        x_prev = xr
        y = to_np(ctx.tf_gn_matvec(d, grams, wt, torch.from_numpy(v).cuda(), lam))
        yr = oracle.gn_matvec_hv(w, v, lam, I, J, K, R)
        mv.append(rel_err(y, yr))
        # per element: 1e-10 of the element or of its block's scale, or the fp64 forward-error bound of the matvec's
        # terms where the result cancels (Jacobi-scaled directions: terms ~1e3 summing to ~1e-4 at c5)
        terms, k = hv_abs_terms(w, v, lam, I, J, K, R)
        check_elementwise_floor(y, yr, blocks, k * U * terms)
    _report(f"cg/{key}", {"x_drift": drift, "r2_rel": r2err, "matvec_rel": mv, "x_bar": x_bar})
    for i, e in enumerate(drift):
        assert e <= x_bar, (key, i + 1, e, drift)
    assert max(r2err) <= 1e-9, (key, r2err)
    assert max(mv) <= TOL
    return drift


@pytest.mark.parametrize("point", ["true", "random"])
@pytest.mark.parametrize("jacobi", [False, True])
def test_c3_cg_per_iteration(ctx, c3, point, jacobi):
    """c3's 10 CG iterations (lambda = 1e-3, rhs = -grad F from the oracle) at full size. Iterate drift bar
    1e-9: the collinear true point's (J^T J + 1e-3 I) has condition number ~1e8, so a 1e-16 rounding
    difference in one matvec grows to ~1e-10..1e-9 in x after 10 iterations in ANY fp64 CG (SURVEY.md §8c
    measured 1.1e-11 at a 60^3 collinear instance); every matvec itself is held to 1e-10."""
    P, ref = c3
    c = P.cfg
    _, gr = ref[point]
    _cg_parity(ctx, f"c3/{point}/jacobi={int(jacobi)}", to_np(P.w(point)), -gr, c.lam, 10, jacobi, c.I, c.J, c.K,
               c.R, 1e-9)


def test_c3_cg_small_grid(ctx, c3):
    """The same CG on a 37-block grid (tf_ctx_set_cg_grid): every block runs several apply items (the
    restage-skip path c5 takes on the full grid), same iterates."""
    P, ref = c3
    c = P.cfg
    _, gr = ref["random"]
    ctx.set_cg_grid(37)
    try:
        _cg_parity(ctx, "c3/random/grid37", to_np(P.w("random")), -gr, c.lam, 10, True, c.I, c.J, c.K, c.R, 1e-9)
    finally:
        ctx.set_cg_grid(0)


# ------------------------------------------------------------------------------ R31 guard boundary (c3)
def _wpi_norm(w, I, J, K, R):
    G = oracle.grams(w, I, J, K, R)
    Pi = oracle.hadamard_chains(G, R)
    RR = R * R
    tot = 0.0
    for l, (off, n) in enumerate(((0, I), (I * R, J), ((I + J) * R, K))):
        Wl = w[off:off + n * R].reshape(R, n).T
        Pl = Pi[l * RR:(l + 1) * RR].reshape(R, R).T
        tot += float(np.linalg.norm(Wl @ Pl)) ** 2
    return math.sqrt(tot)


def test_pi_guard_boundary_c3(ctx, c3):
    """Reading R31 at its thresholds, c3 full size, forced Pi form. Along an A-only direction d the objective is
    exactly quadratic (the model is linear in A): F(w* + t d) = F* + t<grad F*, d> + t^2/2 <d, J^T J d>, so t is
    solved from the oracle's F*, grad F* and Thm-Hv matvec for 2F/||T||^2 = 1.05e-3, 2e-3, 1e-2 (both ratios are
    then measured by the oracle at the chosen point). At SNR 20 dB the true point has 2F/||T||^2 ~ 1e-2 but
    ||grad||/||W Pi|| ~ 2.5e-4 (the gradient guard falls back), and t along d is solved (to first order,
    grad(t) ~ grad* + t J^T J d) for ||grad||/||W Pi|| = 1.1e-3. Every case: no fallback, F and grad within 1e-10
    of the oracle."""
    P, ref = c3
    c = P.cfg
    I, J, K, R = c.I, c.J, c.K, c.R
    nT2 = t_norm2(P.T)
    w0 = to_np(P.w("true"))
    f0, g0 = ref["true"]
    rng = np.random.default_rng(1)
    dvec = np.zeros_like(w0)
    dvec[:I * R] = rng.standard_normal(I * R)
    a2 = 0.5 * float(np.dot(dvec, oracle.gn_matvec_hv(w0, dvec, 0.0, I, J, K, R)))
    a1 = float(np.dot(g0, dvec))
    cases = []
    for target in (1.05e-3, 2e-3, 1e-2):
        cc = f0 - 0.5 * target * nT2
        t = (-a1 + math.sqrt(a1 * a1 - 4 * a2 * cc)) / (2 * a2)
        cases.append((f"rho={target:g}", P, w0 + t * dvec, nT2))
    P20 = synth.make_problem("c3", "cuda", noise_value=20.0)
    nT2_20 = t_norm2(P20.T)
    w20 = to_np(P20.w("true"))
    f20, g20 = oracle_eval_slabs(P20.T, w20, I, J, K, R)
    ratio20 = np.linalg.norm(g20) / _wpi_norm(w20, I, J, K, R)
    assert 2 * f20 / nT2_20 > 1.05e-3 and ratio20 < 1e-3   # the gradient guard is the one that decides here
    h = oracle.gn_matvec_hv(w20, dvec, 0.0, I, J, K, R)
    W = _wpi_norm(w20, I, J, K, R)
    qa, qb, qc = float(h @ h), 2 * float(g20 @ h), float(g20 @ g20) - (1.1e-3 * W) ** 2
    t = (-qb + math.sqrt(qb * qb - 4 * qa * qc)) / (2 * qa)
    cases.append(("gradratio=1.1e-3", P20, w20 + t * dvec, nT2_20))
    out = {}
    for key, PP, w, n2 in cases:
        fr, gr = oracle_eval_slabs(PP.T, w, I, J, K, R)
        rho = 2 * fr / n2
        gratio = np.linalg.norm(gr) / _wpi_norm(w, I, J, K, R)
        assert rho >= 1.04e-3 and gratio >= 1.04e-3, (key, rho, gratio)   # both guards pass, narrowly
        wt = torch.from_numpy(w).cuda()
        check_eval_full(ctx, PP, wt, fr, gr, "pi", expect_fallback=0, key=f"R31/{key}")
        out[key] = {"rho": rho, "grad_ratio": gratio}
    # the 20 dB true point itself: the gradient guard reruns the residual form, still at the bar
    check_eval_full(ctx, P20, P20.w("true"), f20, g20, "pi", expect_fallback=1, key="R31/snr20-true")
    out["snr20-true"] = {"rho": 2 * f20 / nT2_20, "grad_ratio": ratio20}
    _report("R31/points", out)


# ------------------------------------------------------------------------------------------------ c5
@pytest.fixture(scope="module")
def c5():
    P = synth.make_problem("c5", "cuda")
    c = P.cfg
    fr, gr = oracle_eval_slabs(P.T, P.w("random"), c.I, c.J, c.K, c.R)
    return P, fr, gr


def test_c5_full_vector_eval(ctx, c5):
    """c5 (1200^3, R = 100, 13.8 GB) full size: F and all 360 000 gradient entries in the guarded Pi form (the
    bench's default) and the residual form, against the oracle per block and per element."""
    P, fr, gr = c5
    check_eval_full(ctx, P, P.w("random"), fr, gr, "auto", expect_fallback=0, key="c5/random")
    check_eval_full(ctx, P, P.w("random"), fr, gr, "residual", key="c5/random")


def test_c5_cg_per_iteration(ctx, c5):
    """c5's 20 CG iterations (lambda = 1e-3, rhs = -grad F from the oracle), n = 360 000: the configuration the
    bench times (the persistent grid kernel, more apply items than blocks). Random point: well conditioned, the
    iterate drift stays near rounding (bar 1e-10)."""
    P, fr, gr = c5
    c = P.cfg
    _cg_parity(ctx, "c5/random/jacobi=0", to_np(P.w("random")), -gr, c.lam, 20, False, c.I, c.J, c.K, c.R, 1e-10)


@pytest.mark.parametrize("world", [2, 8])
def test_c5_k_shards_sum_to_full_and_oracle(ctx, c5, world):
    """What one rank of an N-GPU run computes at the benchmark's size: the partial [grad | F] of each
    balanced K-shard (k_begin, K_total; dF/dC rows outside the shard exactly zero), summed over the N shards in rank
    order — the all-reduce — equals the single-device evaluation to 1e-12 (only the reduction tree differs) and the
    oracle to 1e-10 per block and element."""
    P, fr, gr = c5
    c = P.cfg
    I, J, K, R = c.I, c.J, c.K, c.R
    w = P.w("random")
    f1, g1 = ctx.tf_cpd_eval(tf.Dims(I, J, K, R), P.T, w)
    f1, g1 = float(f1.item()), to_np(g1)
    fs, gs = 0.0, np.zeros_like(g1)
    for rank in range(world):
        k0, k1 = synth.shard_range(K, rank, world)
        f, g = ctx.tf_cpd_eval(tf.Dims(I, J, k1 - k0, R, K_total=K, k_begin=k0), P.T[k0:k1], w)
        g = to_np(g)
        gC = g[(I + J) * R:].reshape(R, K)
        assert not gC[:, :k0].any() and not gC[:, k1:].any()
        fs += float(f.item())
        gs += g
    assert abs(fs - f1) <= 1e-12 * abs(f1)
    assert rel_err(gs, g1) <= 1e-12
    okf, ef, bf = within([fs], [fr])
    assert okf, (ef, bf)
    per = check_elementwise(gs, gr, w_blocks(I, J, K, R), block_floors(to_np(w), I, J, K, R))
    _report(f"shards/c5/{world}", {"f_rel_vs_single": abs(fs - f1) / abs(f1), "grad_rel_vs_single": rel_err(gs, g1),
                                   "grad_rel_vs_oracle": rel_err(gs, gr), "blocks": per})


def test_c5_cg_per_iteration_jacobi(ctx, c5):
    """c5's 20 CG iterations with the Jacobi preconditioner M = diag(J^T J) + lambda: the
    scaling folded into the row-owned kernel's operands (Pi~ = D Pi D, S~ = S D) at the bench's size. Every matvec
    is held to 1e-10. The iterate drift is bounded by the conditioning, not by 1e-10: J^T J is singular along the
    2R scaling directions of the CPD, which lambda I regularises; in the Jacobi coordinates
    that eigenvalue is lambda D^2 ~ 1e-3 / ||B_r||^2 ||C_r||^2 ~ 7e-10 against O(1) elsewhere, and the scaled
    right-hand side D rhs is not orthogonal to those directions (rhs is, without scaling). So kappa ~ 3 /
    (lambda min D^2) ~ 4e9, and any fp64 CG drifts from the 80-bit oracle by ~u kappa ~ 1e-6 once the
    well-conditioned part has converged (iteration ~13 here); the bar is 10 u kappa_est."""
    P, fr, gr = c5
    c = P.cfg
    w = to_np(P.w("random"))
    I, J, K, R = c.I, c.J, c.K, c.R
    d2 = oracle.jtj_diag(w, I, J, K, R) + c.lam            # M = diag(J^T J) + lambda
    kappa_est = 3.0 / (c.lam / float(d2.max()))
    _cg_parity(ctx, "c5/random/jacobi=1", w, -gr, c.lam, 20, True, I, J, K, R, 10 * U * kappa_est)


def test_c5_host_streamed_eval(ctx, c5):
    """The e2e path at the bench's size: tf_cpd_eval_host streams the 13.8 GB T from pinned host memory in 512 MB
    slabs (K-shards summed on the device); F and the whole gradient against the oracle per block and element."""
    P, fr, gr = c5
    c = P.cfg
    I, J, K, R = c.I, c.J, c.K, c.R
    T_host = torch.empty(P.T.shape, dtype=torch.float64, pin_memory=True)
    T_host.copy_(P.T)
    w_host = P.w("random").cpu().contiguous()
    fh, gh = ctx.tf_cpd_eval_host(tf.Dims(I, J, K, R), T_host, w_host)
    okf, ef, bf = within([float(fh.item())], [fr])
    assert okf, (ef, bf)
    per = check_elementwise(to_np(gh), gr, w_blocks(I, J, K, R), block_floors(to_np(w_host), I, J, K, R))
    _report("eval/c5/host_streamed", {"f_rel": ef / abs(fr), "grad_rel": rel_err(to_np(gh), gr), "blocks": per})


# ------------------------------------------------------------------------------------------------ c4
def test_c4_full_vector_eval(ctx):
    """c4 (4000 x 800 x 400, R = 50, U(0,1) factors) at full size: unequal modes, half-empty edge tiles in I and J,
    the default Pi form and the residual form; F and all 260 000 gradient entries against the oracle per block
    and per element."""
    P = synth.make_problem("c4", "cuda")
    c = P.cfg
    w = P.w("random_uniform")
    fr, gr = oracle_eval_slabs(P.T, w, c.I, c.J, c.K, c.R)
    check_eval_full(ctx, P, w, fr, gr, "auto", expect_fallback=0, key="c4/random_uniform")
    check_eval_full(ctx, P, w, fr, gr, "residual", key="c4/random_uniform")
