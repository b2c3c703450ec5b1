"""Parity of the CUDA path (through the C ABI) with the CPU oracle, element by element.

Bar (north_star): relative error <= 1e-10 in fp64, ‖Δ‖/max(‖ref‖, floor) with the
floors of DESIGN.md reading R14 (active only where the reference is ~0).
"""
import json
import math
import os

import numpy as np
import pytest
import torch

import oracle
import synth
from parity_util import TOL, f_floor, grad_floor, rel_err, to_np, within

pytestmark = pytest.mark.gpu

tf = pytest.importorskip("paper_2110_05997_b200")


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    c = tf.Context(0)
    yield c
    c.close()


def run_eval(ctx, T_t, w_t, I, J, K, R, **kw):
    d = tf.Dims(I, J, K, R, **kw)
    T = T_t.cuda().contiguous()
    w = w_t.cuda().contiguous()
    f, g = ctx.tf_cpd_eval(d, T, w)
    torch.cuda.synchronize()
    return float(f.item()), to_np(g)


def check_eval(ctx, T_np, w_np, I, J, K, R, tol=TOL):
    T_t = torch.from_numpy(np.ascontiguousarray(T_np, dtype=np.float64))
    w_t = torch.from_numpy(np.ascontiguousarray(w_np, dtype=np.float64))
    f, g = run_eval(ctx, T_t, w_t, I, J, K, R)
    fr, gr = oracle.cpd_eval(T_np, w_np, I, J, K, R)
    okf, ef, bf = within([f], [fr], f_floor(T_np, fr), tol)
    okg, eg, bg = within(g, gr, grad_floor(w_np, I, J, K, R), tol)
    assert okf, ("f", ef, bf, f, fr)
    assert okg, ("grad", eg, bg)
    return ef, eg


# ------------------------------------------------------------------------- configs c1, c2 (full oracle)
@pytest.mark.parametrize("point", ["true", "perturbed"])
def test_c1_eval(ctx, point):
    P = synth.make_problem("c1", "cpu")
    c = P.cfg
    check_eval(ctx, to_np(P.T).reshape(-1), to_np(P.w(point)), c.I, c.J, c.K, c.R)


def test_c2_eval(ctx):
    P = synth.make_problem("c2", "cpu")
    c = P.cfg
    check_eval(ctx, to_np(P.T).reshape(-1), to_np(P.w("random")), c.I, c.J, c.K, c.R)


@pytest.mark.parametrize("name,dims", [("c3", (130, 70, 40, 20)), ("c4", (200, 90, 33, 50)),
                                       ("c5", (100, 77, 21, 100))])
def test_reduced_recipes_eval(ctx, name, dims):
    """c3-c5 recipes at sizes the oracle finishes in seconds, spanning several tiles and a ragged tail."""
    P = synth.make_problem(name, "cpu", dims=dims)
    I, J, K, R = dims
    for point, w in P.points.items():
        check_eval(ctx, to_np(P.T).reshape(-1), to_np(w), I, J, K, R)


# ------------------------------------------------------------------------- shapes and edge cases
@pytest.mark.parametrize("dims", [(1, 1, 1, 1), (2, 3, 1, 1), (64, 64, 2, 8), (65, 63, 3, 9), (3, 5, 7, 2),
                                  (7, 129, 5, 4), (128, 1, 2, 16), (20, 20, 20, 128), (66, 70, 4, 104)])
def test_shapes(ctx, dims):
    I, J, K, R = dims
    rng = np.random.default_rng(sum(dims))
    T = rng.standard_normal(I * J * K)
    w = rng.standard_normal(R * (I + J + K))
    check_eval(ctx, T, w, I, J, K, R)


@pytest.mark.parametrize("form", ["residual", "pi"])
@pytest.mark.parametrize("split", ["chunks", "streamk-cps1", "streamk-cps2", "streamk-cps3"])
@pytest.mark.parametrize("dims", [(130, 70, 40, 20), (200, 150, 61, 13), (65, 63, 3, 9), (90, 40, 7, 33)])
def test_eval_work_decompositions(ctx, dims, split, form, monkeypatch):
    """The fused kernel's two decompositions of the (tile, slice) space agree with the oracle: one k-chunk per CTA,
    and stream-K (equal runs of units per CTA of a persistent grid; the runs cut tiles mid-K, so a tile's partials
    come from several segments, and a CTA crosses tile boundaries). The CTAs-per-SM override moves the cut points."""
    if split == "chunks":
        monkeypatch.setenv("TF_EVAL_STREAMK", "0")
    else:
        monkeypatch.setenv("TF_EVAL_PERSIST_CPS", split[-1])
    I, J, K, R = dims
    rng = np.random.default_rng(I * J + K + R)
    T = rng.standard_normal(I * J * K)
    w = rng.standard_normal(R * (I + J + K))
    ctx.set_eval_form(form)
    try:
        check_eval(ctx, T, w, I, J, K, R)
    finally:
        ctx.set_eval_form("auto")


@pytest.mark.parametrize("decouple", ["0", "1", "2"])
@pytest.mark.parametrize("dims", [(130, 70, 40, 20), (200, 150, 61, 13), (90, 40, 7, 33), (52, 52, 19, 100),
                                  (256, 200, 75, 24)])
def test_eval_decoupled_warp_groups(ctx, dims, decouple, monkeypatch):
    """The Pi pass with the per-slice block barrier (0) and with decoupled warp groups (mbarrier hand-offs of T_k
    and c_k, the dF/dC rows and the buffers; 1 throttled, 2 unthrottled) agrees with the oracle, on stream-K runs
    that cross tiles (segments of 1..17 slices, so every issue / wait path of the two-buffer ring runs)."""
    monkeypatch.setenv("TF_EVAL_DECOUPLE", decouple)
    I, J, K, R = dims
    rng = np.random.default_rng(7 * I + J + K + R)
    T = rng.standard_normal(I * J * K)
    w = rng.standard_normal(R * (I + J + K))
    ctx.set_eval_form("pi")
    try:
        check_eval(ctx, T, w, I, J, K, R)
        assert ctx.eval_fell_back() == 0
    finally:
        ctx.set_eval_form("auto")


@pytest.mark.parametrize("form", ["auto", "pi"])
def test_padded_leading_dimension(ctx, form):
    """ldT > I (both an even ldT -> TMA path and an odd ldT -> cooperative-load path), both forms."""
    ctx.set_eval_form(form)
    try:
        _padded_ld(ctx)
    finally:
        ctx.set_eval_form("auto")


def _padded_ld(ctx):
    I, J, K, R = 30, 17, 6, 5
    rng = np.random.default_rng(5)
    t = rng.standard_normal((K, J, I))
    w = rng.standard_normal(R * (I + J + K))
    fr, gr = oracle.cpd_eval(t.reshape(-1), w, I, J, K, R)
    for ldT in (32, 33):
        Tp = np.zeros((K, J, ldT))
        Tp[:, :, :I] = t
        Tp[:, :, I:] = 1e300   # padding must never be read
        Tt = torch.from_numpy(Tp.reshape(-1)).cuda()
        f, g = ctx.tf_cpd_eval(tf.Dims(I, J, K, R, ldT=ldT), Tt, torch.from_numpy(w).cuda())
        assert ctx.eval_used_tma() == (1 if ldT % 2 == 0 else 0)   # the library reports the load path it ran
        assert rel_err([f.item()], [fr]) <= TOL
        assert rel_err(to_np(g), gr) <= TOL


@pytest.mark.parametrize("form", ["residual", "pi"])
@pytest.mark.parametrize("dims", [(50, 40, 23, 6), (40, 40, 23, 6)])
def test_k_sharded_partials_sum_to_full(ctx, form, dims):
    """shard partials [grad | f] summed elementwise equal the full evaluation (both
    algebraic forms of reading R31; in the Pi form each shard uses the C Gram over its own slices; I = J takes
    the batched Gram / W Pi launches)."""
    ctx.set_eval_form(form)
    try:
        _sharded_partials(ctx, *dims)
    finally:
        ctx.set_eval_form("auto")


def _sharded_partials(ctx, I, J, K, R):
    rng = np.random.default_rng(11)
    t = rng.standard_normal((K, J, I))
    w = torch.from_numpy(rng.standard_normal(R * (I + J + K))).cuda()
    Tt = torch.from_numpy(t).cuda()
    f_full, g_full = ctx.tf_cpd_eval(tf.Dims(I, J, K, R), Tt, w)
    grams_full = ctx.tf_grams(tf.Dims(I, J, K, R), w)
    acc_f = torch.zeros(1, dtype=torch.float64, device="cuda")
    acc_g = torch.zeros_like(g_full)
    for world in (2, 3, 5, 8):
        acc_f.zero_()
        acc_g.zero_()
        for rank in range(world):
            k0, k1 = synth.shard_range(K, rank, world)
            grams = torch.empty(3 * R * R, dtype=torch.float64, device="cuda")
            f, g = ctx.tf_cpd_eval(tf.Dims(I, J, k1 - k0, R, K_total=K, k_begin=k0), Tt[k0:k1].contiguous(), w,
                                   grams=grams)
            # the Grams returned with a shard's evaluation are those of the full (replicated) factors
            assert rel_err(to_np(grams), to_np(grams_full)) <= 1e-13
            # rows of dF/dC outside the shard are exactly zero
            gC = g[(I + J) * R:].view(R, K)
            assert torch.all(gC[:, :k0] == 0) and torch.all(gC[:, k1:] == 0)
            acc_f += f
            acc_g += g
        assert rel_err(to_np(acc_f), to_np(f_full)) <= 1e-12
        assert rel_err(to_np(acc_g), to_np(g_full)) <= 1e-12
    fr, gr = oracle.cpd_eval(t.reshape(-1), to_np(w), I, J, K, R)
    assert rel_err(to_np(acc_g), gr) <= TOL


def test_deterministic_bitwise(ctx):
    P = synth.make_problem("c2", "cpu", dims=(96, 80, 50, 10))
    T = P.T.cuda()
    w = P.w("random").cuda()
    d = tf.Dims(96, 80, 50, 10)
    f1, g1 = ctx.tf_cpd_eval(d, T, w)
    f1, g1 = f1.clone(), g1.clone()
    for _ in range(3):
        f2, g2 = ctx.tf_cpd_eval(d, T, w)
        assert torch.equal(f1, f2) and torch.equal(g1, g2)


def test_host_streamed_eval_matches_device(ctx):
    P = synth.make_problem("c2", "cpu", dims=(64, 50, 40, 7))
    d = tf.Dims(64, 50, 40, 7)
    fh, gh = ctx.tf_cpd_eval_host(d, P.T.contiguous(), P.w("random").contiguous())
    fr, gr = oracle.cpd_eval(to_np(P.T).reshape(-1), to_np(P.w("random")), 64, 50, 40, 7)
    assert rel_err(to_np(fh), [fr]) <= TOL
    assert rel_err(to_np(gh), gr) <= TOL


@pytest.mark.slow
def test_host_streamed_eval_c3_full_size(ctx):
    """The e2e path at c3's full size (1 GB: two 512 MB slabs, each a K-shard large enough for the guarded Pi
    form): the streamed result equals the device-resident evaluation to rounding (the slabs' partial sums
    only change the reduction order), and the device one is pinned to the oracle by test_c3_full_size_sampled."""
    P = synth.make_problem("c3", "cuda")
    c = P.cfg
    d = tf.Dims(c.I, c.J, c.K, c.R)
    w = P.w("random")
    fd, gd = ctx.tf_cpd_eval(d, P.T, w)
    torch.cuda.synchronize()
    assert ctx.eval_fell_back() == 0   # the Pi form ran
    fh, gh = ctx.tf_cpd_eval_host(d, P.T.cpu().contiguous(), w.cpu().contiguous())
    assert rel_err(to_np(fh), to_np(fd)) <= 1e-12
    assert rel_err(to_np(gh), to_np(gd)) <= 1e-12


# ------------------------------------------------------------------------- paper fixtures
def _w_of(A, B, C):
    return np.concatenate([A.T.reshape(-1), B.T.reshape(-1), C.T.reshape(-1)])


def test_warmup_fixture(ctx, golden_dir):
    g = json.load(open(os.path.join(golden_dir, "warmup.json")))
    x, y = np.array(g["x"]), np.array(g["y"])
    z = np.array(g["z_num"], dtype=np.float64) / g["z_den"]
    X, Y, Z = np.meshgrid(x, y, z, indexing="ij")
    t = (np.cos(1 - X) * np.sin(1 + Y ** 2) - np.sin(1 + X ** 2) * np.exp(X ** 2 + Y ** 2 + Z ** 2)
         - np.cos(X) * np.log(1 + Z))
    T = np.ascontiguousarray(t.transpose(2, 1, 0)).reshape(-1)
    A = np.stack([np.cos(1 - x), -np.sin(1 + x ** 2) * np.exp(x ** 2), -np.cos(x)], axis=1)
    B = np.stack([np.sin(1 + y ** 2), np.exp(y ** 2), np.ones_like(y)], axis=1)
    C = np.stack([np.ones_like(z), np.exp(z ** 2), np.log(1 + z)], axis=1)
    # at the true factors F and grad are ~0: the bound is the fp64 floor (reading R14)
    check_eval(ctx, T, _w_of(A, B, C), 6, 5, 4, 3)
    # at the paper's printed final CPD
    Xp, Yp, Zp = (np.array(g[k]) for k in ("printed_X", "printed_Y", "printed_Z"))
    check_eval(ctx, T, _w_of(Xp, Yp, Zp), 6, 5, 4, 3)


@pytest.mark.parametrize("n", [10.0, 1000.0])
def test_border_rank_fixture(ctx, n):
    I, J, K = 3, 4, 2
    e = lambda m, k: np.eye(m)[:, k]
    t = (np.einsum("i,j,k->ijk", e(I, 0), e(J, 0), e(K, 1)) + np.einsum("i,j,k->ijk", e(I, 0), e(J, 1), e(K, 0))
         + np.einsum("i,j,k->ijk", e(I, 1), e(J, 0), e(K, 0)))
    A = np.stack([n * (e(I, 0) + e(I, 1) / n), -n * e(I, 0)], axis=1)
    B = np.stack([e(J, 0) + e(J, 1) / n, e(J, 0)], axis=1)
    C = np.stack([e(K, 0) + e(K, 1) / n, e(K, 0)], axis=1)
    T = np.ascontiguousarray(t.transpose(2, 1, 0)).reshape(-1)
    f, _ = run_eval(ctx, torch.from_numpy(T), torch.from_numpy(_w_of(A, B, C)), I, J, K, 2)
    ref = 0.5 * (3.0 / n ** 2 + 1.0 / n ** 4)
    assert abs(f - ref) <= 1e-10 * ref
    check_eval(ctx, T, _w_of(A, B, C), I, J, K, 2)


# ------------------------------------------------------------------------- Grams, Hadamard, matvec, CG
def test_grams_and_hadamard(ctx):
    I, J, K, R = 300, 45, 70, 37
    rng = np.random.default_rng(3)
    w = rng.standard_normal(R * (I + J + K))
    d = tf.Dims(I, J, K, R)
    wt = torch.from_numpy(w).cuda()
    g = ctx.tf_grams(d, wt)
    pi = ctx.tf_hadamard(R, g)
    gr = oracle.grams(w, I, J, K, R)
    assert rel_err(to_np(g), gr) <= TOL
    assert rel_err(to_np(pi), oracle.hadamard_chains(gr, R)) <= TOL
    # grams as the optional output of tf_cpd_eval
    T = torch.from_numpy(rng.standard_normal(I * J * K)).cuda()
    g2 = torch.empty_like(g)
    ctx.tf_cpd_eval(d, T, wt, grams=g2)
    assert torch.equal(g, g2)


@pytest.mark.parametrize("dims", [(20, 20, 20, 3), (200, 200, 200, 10), (500, 300, 40, 20), (120, 80, 60, 100),
                                  (61, 47, 33, 120), (7, 5, 3, 1), (1, 1, 1, 9)])
@pytest.mark.parametrize("lam", [0.0, 1e-3])
def test_gn_matvec(ctx, dims, lam):
    I, J, K, R = dims
    rng = np.random.default_rng(I + R)
    w = rng.standard_normal(R * (I + J + K))
    v = rng.standard_normal(R * (I + J + K))
    d = tf.Dims(I, J, K, R)
    wt = torch.from_numpy(w).cuda()
    g = ctx.tf_grams(d, wt)
    y = ctx.tf_gn_matvec(d, g, wt, torch.from_numpy(v).cuda(), lam)
    ref = oracle.gn_matvec_hv(w, v, lam, I, J, K, R)
    assert rel_err(to_np(y), ref) <= TOL


def test_gn_matvec_against_plain_route(ctx):
    """Against the oracle's J-then-J^T route (no Grams) on c1."""
    P = synth.make_problem("c1", "cpu")
    c = P.cfg
    w = to_np(P.w("perturbed"))
    v = to_np(synth.random_vector(c.n, "cpu", "c1-matvec"))
    d = tf.Dims(c.I, c.J, c.K, c.R)
    wt = torch.from_numpy(w).cuda()
    y = ctx.tf_gn_matvec(d, ctx.tf_grams(d, wt), wt, torch.from_numpy(v).cuda(), 1e-3)
    assert rel_err(to_np(y), oracle.gn_matvec_plain(w, v, 1e-3, c.I, c.J, c.K, c.R)) <= TOL


@pytest.mark.parametrize("kernel", ["auto", "grid"])
@pytest.mark.parametrize("grid", [0, 5])
@pytest.mark.parametrize("jacobi", [False, True])
@pytest.mark.parametrize("case", ["c1", "c3r", "r120", "even30", "even31"])
def test_cg_per_iteration(ctx, case, jacobi, grid, kernel, monkeypatch):
    """Every CG iterate x^(i), i = 1..10, against Alg. CG-dGN in the oracle (rhs = -grad, lambda = 1e-3), through
    both persistent kernels: "auto" (the row-owned kernel wherever its shared memory fits — every case here but
    R = 120 — and the one-CTA kernel for n <= 4096 on the default grid) and "grid" (TF_CG_KERNEL=grid: the
    item-based grid kernel). grid = 5 caps the launch at 5 blocks (tf_ctx_set_cg_grid): the row-owned kernel then
    owns 2-6 m-tiles per block, the grid kernel processes several Gram and apply items per block."""
    if kernel == "grid":
        monkeypatch.setenv("TF_CG_KERNEL", "grid")
    ctx.set_cg_grid(grid)
    try:
        _cg_per_iteration(ctx, case, jacobi)
    finally:
        ctx.set_cg_grid(0)


def _cg_per_iteration(ctx, case, jacobi):
    if case == "c1":
        P = synth.make_problem("c1", "cpu")
        I, J, K, R = 20, 20, 20, 3
        w = to_np(P.w("perturbed"))
    elif case == "c3r":
        P = synth.make_problem("c3", "cpu", dims=(60, 50, 40, 20))
        I, J, K, R = 60, 50, 40, 20
        w = to_np(P.w("random"))
    elif case == "r120":   # R > 104 exercises the 16-row apply tiles of the persistent CG kernel
        P = synth.make_problem("c5", "cpu", dims=(37, 29, 23, 120))
        I, J, K, R = 37, 29, 23, 120
        w = to_np(P.w("random"))
    else:   # n > 4096 with even mode sizes: the grid kernel's 16-byte staging paths (R even: also [Pi; S] pairs)
        I, J, K = 80, 64, 48
        R = 30 if case == "even30" else 31
        P = synth.make_problem("c3", "cpu", dims=(I, J, K, R))
        w = to_np(P.w("random"))
    T = to_np(P.T).reshape(-1)
    _, grad = oracle.cpd_eval(T, w, I, J, K, R)
    rhs = -grad
    lam = 1e-3
    ref = oracle.cg(w, rhs, lam, 10, I, J, K, R, jacobi=jacobi, history=True)
    d = tf.Dims(I, J, K, R)
    wt = torch.from_numpy(w).cuda()
    g = ctx.tf_grams(d, wt)
    rt = torch.from_numpy(rhs).cuda()
    for i in range(1, ref["iters"] + 1):
        x, it, r2 = ctx.tf_cg_solve(d, g, wt, rt, lam, i, 0.0, jacobi)
        assert it == i
        e = rel_err(to_np(x), ref["x_hist"][i - 1])
        assert e <= 1e-9, (i, e)      # CG drift grows with conditioning (SURVEY.md §7 hard part 10)
        assert abs(r2 - ref["r2"][i - 1]) <= 1e-8 * ref["r2"][0]


def test_cg_tolerance_stop(ctx):
    P = synth.make_problem("c1", "cpu")
    I, J, K, R = 20, 20, 20, 3
    w = to_np(P.w("perturbed"))
    _, grad = oracle.cpd_eval(to_np(P.T).reshape(-1), w, I, J, K, R)
    d = tf.Dims(I, J, K, R)
    wt = torch.from_numpy(w).cuda()
    g = ctx.tf_grams(d, wt)
    ref = oracle.cg(w, -grad, 1e-3, 200, I, J, K, R, tol=1e-6)
    x, it, r2 = ctx.tf_cg_solve(d, g, wt, torch.from_numpy(-grad).cuda(), 1e-3, 200, 1e-6, False)
    assert it == ref["iters"] and r2 < 1e-6
    assert rel_err(to_np(x), ref["x"]) <= 1e-8


# ------------------------------------------------------------------------- errors
def test_argument_errors(ctx):
    w = torch.zeros(30, dtype=torch.float64, device="cuda")
    T = torch.zeros(8, dtype=torch.float64, device="cuda")
    with pytest.raises(tf.TfError) as ei:
        ctx.tf_cpd_eval(tf.Dims(2, 2, 2, 0), T, w)
    assert ei.value.status == tf.TF_ERR_ARG
    with pytest.raises(tf.TfError) as ei:
        ctx.tf_cpd_eval(tf.Dims(2, 2, 2, 1, ldT=1), T, w)
    assert ei.value.status == tf.TF_ERR_ARG
    with pytest.raises(tf.TfError) as ei:
        ctx.tf_cpd_eval(tf.Dims(2, 2, 2, 1, K_total=3, k_begin=2), T, w)
    assert ei.value.status == tf.TF_ERR_ARG
    big = torch.zeros(200 * 6, dtype=torch.float64, device="cuda")
    with pytest.raises(tf.TfError) as ei:
        ctx.tf_cpd_eval(tf.Dims(2, 2, 2, 200), T, big)
    assert ei.value.status == tf.TF_ERR_UNSUPPORTED


# ------------------------------------------------------------------------- full sizes, sampled outputs
def _sampled_full_size(ctx, name, point, n_rows=2):
    P = synth.make_problem(name, "cuda")
    c = P.cfg
    I, J, K, R = c.I, c.J, c.K, c.R
    d = tf.Dims(I, J, K, R)
    w = P.w(point)
    f, g = ctx.tf_cpd_eval(d, P.T, w)
    g = to_np(g)
    wn = to_np(w)
    A = wn[:I * R].reshape(R, I).T
    B = wn[I * R:(I + J) * R].reshape(R, J).T
    C = wn[(I + J) * R:].reshape(R, K).T
    gA = g[:I * R].reshape(R, I).T
    gB = g[I * R:(I + J) * R].reshape(R, J).T
    gC = g[(I + J) * R:].reshape(R, K).T
    rng = np.random.default_rng(7)
    scale = float(np.linalg.norm(g))
    for i in list(rng.choice(I, n_rows, replace=False)) + [I - 1]:
        S = P.T[:, :, i].cpu().numpy().T          # (J, K) horizontal slice T[i,:,:]
        _, row = oracle.slice_eval(S, A[i], B, C)
        assert np.linalg.norm(gA[i] - row) <= TOL * max(np.linalg.norm(row), scale / math.sqrt(I))
    for j in list(rng.choice(J, n_rows, replace=False)) + [J - 1]:
        S = P.T[:, j, :].cpu().numpy().T          # (I, K) lateral slice
        _, row = oracle.slice_eval(S, B[j], A, C)
        assert np.linalg.norm(gB[j] - row) <= TOL * max(np.linalg.norm(row), scale / math.sqrt(J))
    ks = list(rng.choice(K, n_rows, replace=False)) + [K - 1]
    for k in ks:
        S = P.T[k].cpu().numpy().T                # (I, J) frontal slice
        fs, row = oracle.slice_eval(S, C[k], A, B)
        assert np.linalg.norm(gC[k] - row) <= TOL * max(np.linalg.norm(row), scale / math.sqrt(K))
        # the objective of one slice through the 1-slice sharded call, in the bench's launch configuration
        f1, _ = ctx.tf_cpd_eval(tf.Dims(I, J, 1, R, K_total=K, k_begin=int(k)), P.T[k:k + 1], w)
        assert abs(f1.item() - fs) <= TOL * fs
    # f = sum of slice objectives (property at any size): compare with the per-slab sharded sum
    parts = []
    for k0 in range(0, K, max(1, K // 7)):
        k1 = min(K, k0 + max(1, K // 7))
        fp, _ = ctx.tf_cpd_eval(tf.Dims(I, J, k1 - k0, R, K_total=K, k_begin=k0), P.T[k0:k1], w)
        parts.append(fp.item())
    assert abs(sum(parts) - f.item()) <= 1e-12 * f.item()


@pytest.mark.slow
def test_c3_full_size_sampled(ctx):
    _sampled_full_size(ctx, "c3", "true")
    _sampled_full_size(ctx, "c3", "random")


@pytest.mark.slow
def test_c4_full_size_sampled(ctx):
    """Unequal modes at full size (4000 x 800 x 400, R = 50): edge tiles in every mode, no batched GEMMs."""
    _sampled_full_size(ctx, "c4", "random_uniform", n_rows=1)


@pytest.mark.slow
def test_c5_full_size_sampled(ctx):
    _sampled_full_size(ctx, "c5", "random", n_rows=1)


# ------------------------------------------------------------------------- NEXT #1: the paper's damping D
def test_reg_gamma(ctx):
    for (I, J, K, R) in [(30, 20, 10, 4), (200, 90, 40, 100), (5, 5, 5, 1)]:
        rng = np.random.default_rng(R)
        w = rng.standard_normal(R * (I + J + K)) * 1.7
        d = tf.Dims(I, J, K, R)
        wt = torch.from_numpy(w).cuda()
        gam = ctx.tf_reg_gamma(R, ctx.tf_grams(d, wt))
        assert rel_err(to_np(gam), oracle.reg_gamma(w, I, J, K, R)) <= TOL


@pytest.mark.parametrize("dims", [(20, 20, 20, 3), (120, 80, 60, 100), (61, 47, 33, 120)])
def test_gn_matvec_damped(ctx, dims):
    I, J, K, R = dims
    rng = np.random.default_rng(I + 3 * R)
    w = rng.standard_normal(R * (I + J + K))
    v = rng.standard_normal(R * (I + J + K))
    d = tf.Dims(I, J, K, R)
    wt = torch.from_numpy(w).cuda()
    g = ctx.tf_grams(d, wt)
    gam = ctx.tf_reg_gamma(R, g)
    y = ctx.tf_gn_matvec_damped(d, g, wt, torch.from_numpy(v).cuda(), 0.37, gam)
    ref = oracle.gn_matvec_hv(w, v, 0.37, I, J, K, R, damp=oracle.reg_gamma(w, I, J, K, R))
    assert rel_err(to_np(y), ref) <= TOL


@pytest.mark.parametrize("jacobi", [False, True])
def test_cg_damped_per_iteration(ctx, jacobi):
    """Alg. CG-dGN on (J^T J + mu D) with Tensor Fox's gamma, every iterate."""
    P = synth.make_problem("c3", "cpu", dims=(60, 50, 40, 20))
    I, J, K, R = 60, 50, 40, 20
    w = to_np(P.w("true"))
    _, grad = oracle.cpd_eval(to_np(P.T).reshape(-1), w, I, J, K, R)
    mu = 0.05
    gam = oracle.reg_gamma(w, I, J, K, R)
    ref = oracle.cg(w, -grad, mu, 8, I, J, K, R, jacobi=jacobi, history=True, damp=gam)
    d = tf.Dims(I, J, K, R)
    wt = torch.from_numpy(w).cuda()
    g = ctx.tf_grams(d, wt)
    gt = ctx.tf_reg_gamma(R, g)
    for i in range(1, ref["iters"] + 1):
        x, it, r2 = ctx.tf_cg_solve_damped(d, g, wt, torch.from_numpy(-grad).cuda(), mu, gt, i, 0.0, jacobi)
        assert it == i
        assert rel_err(to_np(x), ref["x_hist"][i - 1]) <= 1e-9, i


# ------------------------------------------------------------------------- NEXT #2: the dGN outer loop
def _exact_plus_noise(I, J, K, R, seed, sigma):
    rng = np.random.default_rng(seed)
    A, B, C = (rng.standard_normal((n, R)) for n in (I, J, K))
    t = np.einsum("ir,jr,kr->ijk", A, B, C) + sigma * rng.standard_normal((I, J, K))
    T = np.ascontiguousarray(t.transpose(2, 1, 0)).reshape(-1)
    return T, rng.standard_normal(R * (I + J + K))


@pytest.mark.parametrize("use_gamma,jacobi", [(True, True), (False, False)])
def test_dgn_trajectory_matches_oracle(ctx, use_gamma, jacobi):
    """The first dGN iterations (same random CG budgets) match the oracle's iterates: F, mu, g, ||x|| and w."""
    I, J, K, R = 14, 11, 9, 3
    T, w0 = _exact_plus_noise(I, J, K, R, 3, 1e-2)
    cgi = synth.cg_budget(8, seed=4)
    ref = oracle.dgn(T, w0, I, J, K, R, cgi, maxiter=8, tol=0.0, use_gamma=use_gamma, jacobi=jacobi)
    wt = torch.from_numpy(w0.copy()).cuda()
    out, hist = ctx.tf_cpd_dgn(tf.Dims(I, J, K, R), torch.from_numpy(T).cuda(), wt, cgi, maxiter=8, tol=0.0,
                               use_gamma=use_gamma, jacobi=jacobi)
    assert out["iters"] == ref["iters"] >= 5 and out["reason"] == ref["reason"]   # same stop (condition 5 here)
    h, hr = hist, ref["hist"]
    np.testing.assert_array_equal(np.sign(h[:, 3] - 0.25), np.sign(hr[:, 3] - 0.25))   # same damping decisions
    assert rel_err(h[:, 2], hr[:, 2]) <= 1e-12                                      # mu history
    assert rel_err(h[:, 0], hr[:, 0]) <= 1e-8                                       # F history
    assert rel_err(h[:, 4], hr[:, 4]) <= 1e-8                                       # step norms
    assert rel_err(to_np(wt), ref["w"]) <= 1e-8


def test_dgn_converges_on_exact_rank_tensor(ctx):
    """Full run to a stopping condition on an exactly rank-3 tensor: same stop as the oracle, converged fit."""
    I, J, K, R = 9, 8, 7, 3
    T, w0 = _exact_plus_noise(I, J, K, R, 5, 0.0)
    cgi = synth.cg_budget(200, seed=1)
    ref = oracle.dgn(T, w0, I, J, K, R, cgi, tol=1e-6)
    wt = torch.from_numpy(w0.copy()).cuda()
    out, hist = ctx.tf_cpd_dgn(tf.Dims(I, J, K, R), torch.from_numpy(T).cuda(), wt, cgi, tol=1e-6)
    assert out["reason"] == ref["reason"] and out["iters"] == ref["iters"], (out, ref["reason"], ref["iters"])
    assert out["rel_err"] < 1e-5
    assert abs(out["rel_err"] - ref["hist"][-1, 1]) <= 1e-6 * ref["hist"][-1, 1] + 1e-12
    f, _ = oracle.cpd_eval(T, to_np(wt), I, J, K, R)
    assert abs(f - out["f"]) <= 1e-6 * f + 1e-24


# ------------------------------------------------------------------------- guarded Pi-form evaluation (R31)
@pytest.mark.parametrize("case", ["c1-true", "c1-perturbed", "c2", "c3-true", "c3-random", "c4", "c5", "sharded",
                                  "warmup"])
def test_pi_form_and_residual_form_both_match_oracle(ctx, case, golden_dir):
    """tf_cpd_eval in the guarded Pi form (default) and the residual form give the oracle's F and grad within the
    bar; the guard falls back to the residual form exactly where the Gram expansion cancels (near exact fits)
    and keeps the Pi form elsewhere."""
    kw = {}
    if case.startswith("c1"):
        P = synth.make_problem("c1", "cpu")
        point = case.split("-")[1]
    elif case == "c2":
        P, point = synth.make_problem("c2", "cpu"), "random"
    elif case.startswith("c3"):
        P = synth.make_problem("c3", "cpu", dims=(70, 66, 33, 20))
        point = case.split("-")[1]
    elif case == "c4":
        P, point = synth.make_problem("c4", "cpu", dims=(150, 80, 40, 50)), "random_uniform"
    elif case == "c5":
        P, point = synth.make_problem("c5", "cpu", dims=(100, 77, 21, 100)), "random"
    elif case == "sharded":
        P, point = synth.make_problem("c2", "cpu", dims=(64, 70, 50, 10)), "random"
    if case == "warmup":
        g = json.load(open(os.path.join(golden_dir, "warmup.json")))
        x, y = np.array(g["x"]), np.array(g["y"])
        z = np.array(g["z_num"], dtype=np.float64) / g["z_den"]
        X, Y, Z = np.meshgrid(x, y, z, indexing="ij")
        t = (np.cos(1 - X) * np.sin(1 + Y ** 2) - np.sin(1 + X ** 2) * np.exp(X ** 2 + Y ** 2 + Z ** 2)
             - np.cos(X) * np.log(1 + Z))
        T_np = np.ascontiguousarray(t.transpose(2, 1, 0)).reshape(-1)
        A = np.stack([np.cos(1 - x), -np.sin(1 + x ** 2) * np.exp(x ** 2), -np.cos(x)], axis=1)
        B = np.stack([np.sin(1 + y ** 2), np.exp(y ** 2), np.ones_like(y)], axis=1)
        C = np.stack([np.ones_like(z), np.exp(z ** 2), np.log(1 + z)], axis=1)
        w_np = np.concatenate([A.T.reshape(-1), B.T.reshape(-1), C.T.reshape(-1)])
        I, J, K, R = 6, 5, 4, 3
        expect_fallback = 1
    else:
        c = P.cfg
        I, J, K, R = c.I, c.J, c.K, c.R
        T_np, w_np = to_np(P.T).reshape(-1), to_np(P.w(point))
        expect_fallback = 1 if point == "true" else 0
    fr, gr = oracle.cpd_eval(T_np, w_np, I, J, K, R)
    T_t = torch.from_numpy(T_np).cuda()
    w_t = torch.from_numpy(w_np).cuda()
    for form in ("pi", "residual"):
        ctx.set_eval_form(form)
        if case == "sharded":
            f, g = 0.0, np.zeros_like(gr)
            for k0, k1 in ((0, 17), (17, 40), (40, K)):
                d = tf.Dims(I, J, k1 - k0, R, K_total=K, k_begin=k0)
                fp, gp = ctx.tf_cpd_eval(d, T_t.reshape(K, J, I)[k0:k1].contiguous(), w_t)
                f += fp.item()
                g += to_np(gp)
        else:
            fd, gd = ctx.tf_cpd_eval(tf.Dims(I, J, K, R), T_t, w_t)
            f, g = fd.item(), to_np(gd)
        if form == "pi" and case != "sharded":
            assert ctx.eval_fell_back() == expect_fallback, (case, form)
        okf, ef, bf = within([f], [fr], f_floor(T_np, fr))
        okg, eg, bg = within(g, gr, grad_floor(w_np, I, J, K, R))
        assert okf and okg, (case, form, ef, bf, eg, bg)
    ctx.set_eval_form("auto")


# ------------------------------------------------------------------------- K-sharded dGN loop (hook exchange)
def test_sharded_dgn_matches_single_device(ctx):
    """tf_cpd_dgn_sharded on 3 K-shards (3 host threads with their own contexts and streams on this GPU; the
    all-reduce hook sums the ranks' buffers on the host side, no kernel waits on another) follows the
    single-device loop: same iterations and stop, F history and final w to rounding (only the reduction
    order of the partial [grad | F] differs)."""
    import threading
    I, J, K, R = 14, 11, 12, 3
    T, w0 = _exact_plus_noise(I, J, K, R, 7, 1e-2)
    cgi = synth.cg_budget(30, seed=5)
    wt = torch.from_numpy(w0.copy()).cuda()
    ref, href = ctx.tf_cpd_dgn(tf.Dims(I, J, K, R), torch.from_numpy(T).cuda(), wt, cgi, maxiter=30, tol=1e-10)
    world = 3
    Tt = torch.from_numpy(T).reshape(K, J, I)
    bufs = [None] * world
    outs = [None] * world
    barrier = threading.Barrier(world)
    from paper_2110_05997_b200.dist import shard_range

    def run(rank):
        torch.cuda.set_device(0)
        stream = torch.cuda.Stream()
        with torch.cuda.stream(stream):
            c = tf.Context(0, stream)
            k0, k1 = shard_range(K, rank, world)
            Tl = Tt[k0:k1].contiguous().cuda()
            wl = torch.from_numpy(w0.copy()).cuda()
            torch.cuda.synchronize()

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

            out, hist = c.tf_cpd_dgn_sharded(tf.Dims(I, J, k1 - k0, R, K_total=K, k_begin=k0), Tl, wl, cgi, hook,
                                             maxiter=30, tol=1e-10)
            torch.cuda.synchronize()
            outs[rank] = (out, hist, to_np(wl))
            c.close()

    ths = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    for r in range(world):
        out, hist, wr = outs[r]
        assert out["iters"] == ref["iters"] and out["reason"] == ref["reason"], (out, ref)
        n0 = min(8, len(hist))
        assert np.allclose(hist[:n0, 0], href[:n0, 0], rtol=1e-10, atol=0)
        assert np.array_equal(wr, outs[0][2])                       # every rank holds the same w
        assert np.linalg.norm(wr - to_np(wt)) <= 1e-6 * np.linalg.norm(to_np(wt))


@pytest.mark.parametrize("dims", [(37, 29, 23, 1), (37, 29, 23, 5), (70, 66, 40, 9), (64, 64, 17, 33),
                                  (45, 80, 30, 104), (30, 40, 25, 128), (130, 70, 20, 57),
                                  (41, 41, 41, 13), (52, 52, 19, 100)])
def test_pi_form_shapes(ctx, dims):
    """The guarded Pi-form pass forced at every fragment-count regime (R = 1 .. 128: tensor-memory A fragments in
    32 .. 512 columns, two CTAs per SM for R <= 24, R = 128 filling all 512 TMEM columns), ragged tiles, at a
    random point (no fallback): F and grad against the oracle."""
    I, J, K, R = dims
    P = synth.make_problem("c2", "cpu", dims=dims)
    T_np, w_np = to_np(P.T).reshape(-1), to_np(P.w("random"))
    fr, gr = oracle.cpd_eval(T_np, w_np, I, J, K, R)
    ctx.set_eval_form("pi")
    try:
        fd, gd = ctx.tf_cpd_eval(tf.Dims(I, J, K, R), torch.from_numpy(T_np).cuda(), torch.from_numpy(w_np).cuda())
        torch.cuda.synchronize()
        assert ctx.eval_fell_back() == 0
    finally:
        ctx.set_eval_form("auto")
    okf, ef, bf = within([fd.item()], [fr], f_floor(T_np, fr))
    okg, eg, bg = within(to_np(gd), gr, grad_floor(w_np, I, J, K, R))
    assert okf and okg, (dims, ef, bf, eg, bg)


# ------------------------------------------------------------------------- degenerate points
@pytest.mark.parametrize("form", ["residual", "pi"])
@pytest.mark.parametrize("case", ["w_zero", "T_zero", "zero_columns", "rank_one_T"])
def test_degenerate_points(ctx, form, case):
    """Degenerate inputs in both algebraic forms against the oracle: all factors zero (F = 1/2 ||T||^2, grad = 0:
    W Pi and the MTTKRPs both vanish), T = 0 (F = 1/2 ||[[W]]||^2, grad = W Pi), one zero column per factor
    (singular Grams), and an exactly rank-one T evaluated at R = 4 with a perturbed copy of its factor."""
    I, J, K, R = 33, 27, 19, 4
    rng = np.random.default_rng(3)
    T = rng.standard_normal((K, J, I))
    w = rng.standard_normal(R * (I + J + K))
    if case == "w_zero":
        w[:] = 0.0
    elif case == "T_zero":
        T[:] = 0.0
    elif case == "zero_columns":
        for off, nl in ((0, I), (I * R, J), ((I + J) * R, K)):
            w[off + nl * 2: off + nl * 3] = 0.0   # column r = 2 of every factor (w is [vec A | vec B | vec C])
    elif case == "rank_one_T":
        a, b, c = rng.standard_normal(I), rng.standard_normal(J), rng.standard_normal(K)
        T = np.einsum("k,j,i->kji", c, b, a)
        w = 0.1 * rng.standard_normal(R * (I + J + K))
        w[0:I], w[I * R:I * R + J], w[(I + J) * R:(I + J) * R + K] = a, b, c
    ctx.set_eval_form(form)
    try:
        check_eval(ctx, T.reshape(-1), w, I, J, K, R)
    finally:
        ctx.set_eval_form("auto")
    if case == "w_zero":   # exact values, not only the oracle's
        f, g = ctx.tf_cpd_eval(tf.Dims(I, J, K, R), torch.from_numpy(T.reshape(-1)).cuda(), torch.from_numpy(w).cuda())
        assert abs(f.item() - 0.5 * float(np.sum(T * T))) <= 1e-13 * float(np.sum(T * T))
        assert torch.count_nonzero(g).item() == 0


@pytest.mark.parametrize("dims", [(6, 5, 4, 3), (60, 50, 40, 9)])   # the single-CTA and the grid CG kernels
def test_cg_zero_rhs(ctx, dims):
    """Reading R33: rhs = 0 returns x = 0 after zero iterations (no 0/0), like the oracle."""
    I, J, K, R = dims
    n = R * (I + J + K)
    rng = np.random.default_rng(9)
    w = torch.from_numpy(rng.standard_normal(n)).cuda()
    d = tf.Dims(I, J, K, R)
    grams = ctx.tf_grams(d, w)
    x = torch.full((n,), 7.0, dtype=torch.float64, device="cuda")
    for jacobi in (False, True):
        _, iters, r2 = ctx.tf_cg_solve(d, grams, w, torch.zeros(n, dtype=torch.float64, device="cuda"), 1e-3, 10, 0.0,
                                       jacobi, x)
        assert iters == 0 and r2 == 0.0
        assert torch.count_nonzero(x).item() == 0
        ref = oracle.cg(to_np(w), np.zeros(n), 1e-3, 10, I, J, K, R, jacobi=jacobi)
        assert ref["iters"] == 0 and ref["status"] == 0


@pytest.mark.parametrize("jacobi", [False, True])
def test_dgn_cg_breakdown_leaves_w(ctx, jacobi):
    """Stop reason 8 (non-finite CG alpha/beta): a NaN entry in T makes F, grad F and mu^(0) = mean|T| NaN, so
    Alg. CG-dGN meets alpha = NaN at its first iteration. Like the oracle, the loop stops at w^(k-1): w is
    returned bitwise unchanged (no step, no balancing), 0 iterations done, reason 8."""
    I, J, K, R = 14, 11, 9, 3
    T, w0 = _exact_plus_noise(I, J, K, R, 8, 1e-2)
    T[17] = np.nan
    cgi = synth.cg_budget(5, seed=2)
    ref = oracle.dgn(T, w0, I, J, K, R, cgi, maxiter=5, tol=1e-6, jacobi=jacobi)
    assert ref["reason"] == 8 and ref["iters"] == 0 and np.array_equal(ref["w"], w0)
    wt = torch.from_numpy(w0.copy()).cuda()
    out, _ = ctx.tf_cpd_dgn(tf.Dims(I, J, K, R), torch.from_numpy(T).cuda(), wt, cgi, maxiter=5, tol=1e-6,
                            jacobi=jacobi)
    assert out["reason"] == 8 and out["iters"] == 0, out
    assert np.array_equal(to_np(wt), w0)


@pytest.mark.parametrize("case", ["step", "gradient", "divergence"])
def test_dgn_stop_conditions_match_oracle(ctx, case):
    """The dGN loop on the device stops with the same condition at the same iteration as the oracle in the
    constructed runs of tests/test_oracle_pins.py::test_dgn_stops_in_runs (conditions 2, 4 and 7 at k = 1;
    PAPER.md:2756-2773), and returns the same w."""
    I, J, K, R = 5, 4, 3, 2
    rng = np.random.default_rng(31)
    A, B, C = (rng.standard_normal((n, R)) for n in (I, J, K))
    t = np.einsum("ir,jr,kr->ijk", A, B, C) + 0.1 * rng.standard_normal((I, J, K))
    T = np.ascontiguousarray(t.transpose(2, 1, 0)).reshape(-1)
    nT = float(np.linalg.norm(T))
    cgi = np.full(5, 4, dtype=np.int32)
    kw = {}
    if case == "step":
        w0, tol, kw = np.zeros(R * (I + J + K)), 1e-8, {"use_gamma": False, "jacobi": False}
        want = 2
    elif case == "gradient":
        s = 1e-9
        T = T * s
        w0, tol, want = rng.standard_normal(R * (I + J + K)) * s ** (1 / 3), 1e-4, 4
    else:
        T = T / (2 * nT)
        w0, tol, want = 30.0 * rng.standard_normal(R * (I + J + K)), 1.0, 7
    ref = oracle.dgn(T, w0, I, J, K, R, cgi, maxiter=5, tol=tol, **kw)
    assert ref["reason"] == want and ref["iters"] == 1
    wt = torch.from_numpy(w0.copy()).cuda()
    out, _ = ctx.tf_cpd_dgn(tf.Dims(I, J, K, R), torch.from_numpy(T).cuda(), wt, cgi, maxiter=5, tol=tol, **kw)
    assert out["reason"] == want and out["iters"] == 1, out
    assert rel_err(to_np(wt), ref["w"]) <= 1e-9
