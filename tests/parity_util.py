"""Shared helpers for the parity tests (tests only).

Parity bar (north_star + DESIGN.md reading R14): for a GPU output g and the oracle's
g_ref (80-bit), ‖g − g_ref‖₂ ≤ 1e-10·‖g_ref‖₂ + κ·floor with κ = 16, where floor is the
forward-error scale of ANY fp64 evaluation of the residual (u = 2⁻⁵³):
  grad:  u·Σ_ℓ‖W_ℓ Π^(ℓ)‖_F   (residual entries carry ~u·|t_ijk| rounding; contracted with the factors)
  f:     u·‖T‖·sqrt(2 f_ref) + u²‖T‖²
The floor only matters at (near-)exact fits, where the relative error of an fp64
residual is ~u‖T‖/‖E‖ ≫ 1e-10 for every fp64 method; elsewhere the bar is 1e-10 relative.
"""
from __future__ import annotations

import math

import numpy as np
import torch

U = 2.0 ** -53
TOL = 1e-10   # north_star: GPU path within 1e-10 relative of the oracle (fp64)
KAPPA = 16.0


def rel_err(got, ref, floor: float = 0.0) -> float:
    got = np.asarray(got, dtype=np.float64).reshape(-1)
    ref = np.asarray(ref, dtype=np.float64).reshape(-1)
    den = max(float(np.linalg.norm(ref)), floor)
    if den == 0.0:
        return float(np.linalg.norm(got - ref))
    return float(np.linalg.norm(got - ref)) / den


def within(got, ref, floor: float = 0.0, tol: float = TOL):
    """(ok, err, bound) for ‖got − ref‖ ≤ tol‖ref‖ + κ·floor."""
    got = np.asarray(got, dtype=np.float64).reshape(-1)
    ref = np.asarray(ref, dtype=np.float64).reshape(-1)
    err = float(np.linalg.norm(got - ref))
    bound = tol * float(np.linalg.norm(ref)) + KAPPA * floor
    return err <= bound, err, bound


def grad_floor(w, I, J, K, R) -> float:
    w = np.asarray(w, dtype=np.float64).reshape(-1)
    A = w[:I * R].reshape(R, I).T
    B = w[I * R:(I + J) * R].reshape(R, J).T
    C = w[(I + J) * R:].reshape(R, K).T
    gA, gB, gC = A.T @ A, B.T @ B, C.T @ C
    return U * (np.linalg.norm(A @ (gB * gC)) + np.linalg.norm(B @ (gA * gC)) + np.linalg.norm(C @ (gA * gB)))


def f_floor(T, f_ref: float) -> float:
    t = np.asarray(T, dtype=np.float64)
    nT = math.sqrt(float(np.sum(t * t)))
    return U * nT * math.sqrt(2.0 * max(f_ref, 0.0)) + (U * nT) ** 2


def to_np(x) -> np.ndarray:
    if isinstance(x, torch.Tensor):
        return x.detach().cpu().numpy().astype(np.float64)
    return np.asarray(x, dtype=np.float64)


def w_blocks(I, J, K, R):
    """(name, slice) of the three factor blocks of a packed w-layout vector [vec A | vec B | vec C]."""
    return [("A", slice(0, I * R)), ("B", slice(I * R, (I + J) * R)), ("C", slice((I + J) * R, (I + J + K) * R))]


def block_floors(w, I, J, K, R):
    """Per-block forward-error floors u·‖W_ℓ Π^(ℓ)‖_F of an fp64 gradient (reading R14, split by block)."""
    w = np.asarray(w, dtype=np.float64).reshape(-1)
    A = w[:I * R].reshape(R, I).T
    B = w[I * R:(I + J) * R].reshape(R, J).T
    C = w[(I + J) * R:].reshape(R, K).T
    gA, gB, gC = A.T @ A, B.T @ B, C.T @ C
    return [U * np.linalg.norm(A @ (gB * gC)), U * np.linalg.norm(B @ (gA * gC)), U * np.linalg.norm(C @ (gA * gB))]


def check_elementwise(got, ref, blocks, floors=None, tol: float = TOL):
    """Per-block and per-element parity next to the whole-vector norm check.

    For every block b (e.g. dF/dA, dF/dB, dF/dC):
      ‖Δ_b‖₂ ≤ tol·‖ref_b‖₂ + κ·floor_b                                    (a small block cannot hide)
      |Δ_e| ≤ tol·(|ref_e| + rms(ref_b)) + κ·floor_b   for every element e   (nor a single entry)
    rms(ref_b) = ‖ref_b‖₂/√n_b is the block's own scale: an entry far below it (cancellation in its
    contraction) is held to 1e-10 of the block scale, every other entry to 1e-10 of itself.
    Returns a dict of the worst ratios err/bound (≤ 1 passes) per block; raises AssertionError on failure."""
    got = np.asarray(got, dtype=np.float64).reshape(-1)
    ref = np.asarray(ref, dtype=np.float64).reshape(-1)
    out = {}
    for bi, (name, sl) in enumerate(blocks):
        g, r = got[sl], ref[sl]
        if r.size == 0:
            continue
        fl = KAPPA * (floors[bi] if floors is not None else 0.0)
        d = np.abs(g - r)
        nb = float(np.linalg.norm(r))
        blk_bound = tol * nb + fl
        blk_err = float(np.linalg.norm(g - r))
        rms = nb / math.sqrt(r.size)
        el_bound = tol * (np.abs(r) + rms) + fl
        el_ratio = d / np.where(el_bound > 0, el_bound, np.inf)
        worst = int(np.argmax(el_ratio)) if el_ratio.size else 0
        out[name] = {"block_err": blk_err / max(nb, 1e-300), "block_ratio": blk_err / blk_bound if blk_bound > 0 else
                     (0.0 if blk_err == 0 else np.inf), "elem_ratio": float(el_ratio[worst]), "elem_index": worst}
        assert blk_err <= blk_bound, (name, "block", blk_err, blk_bound)
        assert np.all(d <= el_bound), (name, "element", worst, float(g[worst]), float(r[worst]), float(el_bound[worst]))
    return out


def hv_abs_terms(w, v, lam, I, J, K, R):
    """Per element, the sum of the absolute values of every term of (J^T J + lam I) v evaluated by Thm Hv
    (PAPER.md:2352-2370): |V_l| |Pi^(l)| + |W_l| |S_l| + lam |V_l| with |Pi| and |S| built from the absolute Grams
    |W|^T |W| and |V|^T |W|. Any fp64 evaluation order of the matvec (Grams over n_l rows, then 2R-term sums)
    has a forward error of at most (n_max + 2R + 2) u times this per element (the standard dot-product bound), which
    is the element floor where the result cancels (a Jacobi-scaled CG direction at c5: terms ~1e3, entries ~1e-4)."""
    w = np.asarray(w, dtype=np.float64).reshape(-1)
    v = np.asarray(v, dtype=np.float64).reshape(-1)
    dims = (I, J, K)
    offs = (0, I * R, (I + J) * R)
    Wa = [np.abs(w[o:o + n * R].reshape(R, n).T) for o, n in zip(offs, dims)]
    Va = [np.abs(v[o:o + n * R].reshape(R, n).T) for o, n in zip(offs, dims)]
    ga = [X.T @ X for X in Wa]
    gv = [Va[l].T @ Wa[l] for l in range(3)]
    out = []
    for l in range(3):
        o1, o2 = [m for m in range(3) if m != l]
        Pl = ga[o1] * ga[o2]
        # Pi^(l,l') is the Gram of the remaining mode
        Sl = ga[o2] * gv[o1] + ga[o1] * gv[o2]
        out.append((Va[l] @ Pl + Wa[l] @ Sl + abs(lam) * Va[l]).T.reshape(-1))
    return np.concatenate(out), max(dims) + 2 * R + 2


def check_elementwise_floor(got, ref, blocks, elem_floor, tol: float = TOL):
    """check_elementwise with a per-element floor array (e.g. the forward-error bound of hv_abs_terms) in place of
    the per-block one: |Δ_e| ≤ tol·(|ref_e| + rms(ref_b)) + floor_e, and per block ‖Δ_b‖ ≤ tol‖ref_b‖ + ‖floor_b‖."""
    got = np.asarray(got, dtype=np.float64).reshape(-1)
    ref = np.asarray(ref, dtype=np.float64).reshape(-1)
    fl = np.asarray(elem_floor, dtype=np.float64).reshape(-1)
    out = {}
    for name, sl in blocks:
        g, r, f = got[sl], ref[sl], fl[sl]
        if r.size == 0:
            continue
        d = np.abs(g - r)
        nb = float(np.linalg.norm(r))
        blk_bound = tol * nb + float(np.linalg.norm(f))
        blk_err = float(np.linalg.norm(g - r))
        el_bound = tol * (np.abs(r) + nb / math.sqrt(r.size)) + f
        ratio = d / np.where(el_bound > 0, el_bound, np.inf)
        worst = int(np.argmax(ratio))
        out[name] = {"block_ratio": blk_err / blk_bound if blk_bound > 0 else 0.0, "elem_ratio": float(ratio[worst])}
        assert blk_err <= blk_bound, (name, "block", blk_err, blk_bound)
        assert np.all(d <= el_bound), (name, "element", worst, float(g[worst]), float(r[worst]), float(el_bound[worst]))
    return out
