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
