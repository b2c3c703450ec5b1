"""Out-of-bounds and race checks of the CUDA path without compute-sanitizer (closed on this GPU pool).

Every C-ABI call runs with its inputs embedded in NaN guard bands (a read past either end of an input poisons the
result) and its outputs embedded in sentinel bands (a write past either end changes a sentinel), and its outputs
must be bitwise equal to those of the same call on plain, unguarded buffers (the kernels reduce in a fixed order:
equal bits rerun after rerun also rule out shared-memory races that change results). Covered: the fused evaluation
in both algebraic forms on the TMA path (16-byte aligned T) and the cooperative-load path (8-byte aligned T), the
GN matvec, CG through the row-owned, grid and one-CTA kernels, and the dGN loop (w updated in place).
"""
import os

import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu

tf = pytest.importorskip("paper_2110_05997_b200")

G = 4096                       # guard doubles on each side (32 KB: keeps 16-byte alignment)
SENT = 1.2345678901234567e300  # output sentinel


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    c = tf.Context(0)
    yield c
    c.close()


def _guarded(x: torch.Tensor, fill: float, shift: int = 0):
    """(buffer, view): x copied into the middle of a float64 CUDA buffer whose other entries are `fill`; `shift`
    moves the view by that many doubles (shift = 1 -> only 8-byte aligned)."""
    n = x.numel()
    big = torch.full((n + 2 * G + shift,), fill, dtype=torch.float64, device="cuda")
    view = big[G + shift:G + shift + n]
    view.copy_(x.reshape(-1))
    return big, view


def _bands_intact(big: torch.Tensor, n: int, fill: float, shift: int = 0) -> bool:
    lo, hi = big[:G + shift], big[G + shift + n:]
    if np.isnan(fill):
        return bool(torch.isnan(lo).all() and torch.isnan(hi).all())
    return bool((lo == fill).all() and (hi == fill).all())


@pytest.mark.parametrize("form", ["residual", "pi"])
@pytest.mark.parametrize("shift", [0, 1])
@pytest.mark.parametrize("dims", [(20, 20, 20, 3), (65, 63, 3, 9), (130, 70, 40, 20), (45, 80, 30, 104)])
def test_eval_guard_bands(ctx, dims, shift, form):
    I, J, K, R = dims
    P = synth.make_problem("c2", "cpu", dims=dims)
    T = P.T.cuda().contiguous().reshape(-1)
    w = P.w("random").cuda().contiguous()
    d = tf.Dims(I, J, K, R)
    ctx.set_eval_form(form)
    try:
        f0, g0 = ctx.tf_cpd_eval(d, T, w)
        f0, g0 = f0.clone(), g0.clone()
        Tb, Tv = _guarded(T, float("nan"), shift)
        wb, wv = _guarded(w, float("nan"))
        fb, fv = _guarded(torch.zeros(1, dtype=torch.float64), SENT)
        gb, gv = _guarded(torch.zeros(d.n, dtype=torch.float64), SENT)
        ctx.tf_cpd_eval(d, Tv, wv, fv, gv)
        torch.cuda.synchronize()
        assert ctx.eval_used_tma() == (1 if shift == 0 and I % 2 == 0 else 0)   # TMA needs 16-byte T and even ldT
    finally:
        ctx.set_eval_form("auto")
    assert _bands_intact(fb, 1, SENT) and _bands_intact(gb, d.n, SENT)
    assert _bands_intact(Tb, T.numel(), float("nan"), shift) and _bands_intact(wb, d.n, float("nan"))
    assert torch.equal(fv, f0) and torch.equal(gv, g0)


@pytest.mark.parametrize("kernel", ["auto", "grid"])
@pytest.mark.parametrize("dims", [(20, 20, 20, 3), (200, 90, 60, 20), (120, 80, 60, 100), (61, 47, 33, 120)])
def test_cg_and_matvec_guard_bands(ctx, dims, kernel, monkeypatch):
    """The one-CTA kernel (n <= 4096 on the default grid), the row-owned kernel and (TF_CG_KERNEL=grid, or R = 120
    where the row-owned kernel does not fit) the item-based grid kernel, with and without Jacobi scaling."""
    if kernel == "grid":
        monkeypatch.setenv("TF_CG_KERNEL", "grid")
    I, J, K, R = dims
    rng = np.random.default_rng(I + R)
    n = R * (I + J + K)
    w = torch.from_numpy(rng.standard_normal(n)).cuda()
    rhs = torch.from_numpy(rng.standard_normal(n)).cuda()
    d = tf.Dims(I, J, K, R)
    grams = ctx.tf_grams(d, w)
    wb, wv = _guarded(w, float("nan"))
    rb, rv = _guarded(rhs, float("nan"))
    gmb, gmv = _guarded(grams, float("nan"))
    y0 = ctx.tf_gn_matvec(d, grams, w, rhs, 1e-3).clone()
    yb, yv = _guarded(torch.zeros(n, dtype=torch.float64), SENT)
    ctx.tf_gn_matvec(d, gmv, wv, rv, 1e-3, yv)
    torch.cuda.synchronize()
    assert _bands_intact(yb, n, SENT) and torch.equal(yv, y0)
    for jacobi in (False, True):
        x0, it0, r0 = ctx.tf_cg_solve(d, grams, w, rhs, 1e-3, 8, 0.0, jacobi)
        x0 = x0.clone()
        xb, xv = _guarded(torch.zeros(n, dtype=torch.float64), SENT)
        _, it1, r1 = ctx.tf_cg_solve(d, gmv, wv, rv, 1e-3, 8, 0.0, jacobi, xv)
        torch.cuda.synchronize()
        assert _bands_intact(xb, n, SENT), (dims, kernel, jacobi)
        assert it1 == it0 == 8 and r1 == r0 and torch.equal(xv, x0), (dims, kernel, jacobi)
    for buf, cnt in ((wb, n), (rb, n), (gmb, 3 * R * R)):
        assert _bands_intact(buf, cnt, float("nan"))


def test_dgn_guard_bands(ctx):
    """The dGN loop updates w in place: the bands around w (and around T) stay intact, same result as unguarded."""
    I, J, K, R = 30, 25, 20, 4
    P = synth.make_problem("c2", "cpu", dims=(I, J, K, R))
    T = P.T.cuda().contiguous().reshape(-1)
    w0 = P.w("random").cuda().contiguous()
    d = tf.Dims(I, J, K, R)
    cgi = synth.cg_budget(6, seed=1)
    wa = w0.clone()
    ra, ha = ctx.tf_cpd_dgn(d, T, wa, cgi, maxiter=6, tol=0.0)
    Tb, Tv = _guarded(T, float("nan"))
    wb, wv = _guarded(w0, SENT)
    rb_, hb = ctx.tf_cpd_dgn(d, Tv, wv, cgi, maxiter=6, tol=0.0)
    torch.cuda.synchronize()
    assert _bands_intact(wb, d.n, SENT) and _bands_intact(Tb, T.numel(), float("nan"))
    assert torch.equal(wv, wa) and ra == rb_ and np.array_equal(ha, hb)
