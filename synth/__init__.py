"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module is NOT part of the method. It holds no step of the hot path (no
residual, no gradient, no Gram, no matvec, no CG): it only draws random factor
matrices, assembles the input tensor of each workload recipe, and packs/unpacks
the parameter vector layout. Both `oracle/` (through the tests) and the CUDA
path (through the tests and `bench.py`) consume its outputs; neither imports
the other.

Layouts (SURVEY.md §8 notation; PAPER.md:857-872 Alg. Unfolding, 1466-1473):
  * T is I×J×K, fp64, first index fastest: T[i + I*(j + J*k)]. In torch we hold
    it as a contiguous tensor of shape (K, J, I), so T_t[k, j, i] = t_ijk and
    every frontal slice T[:, :, k] is one contiguous column-major I×J block.
  * Factor matrices A (I×R), B (J×R), C (K×R) are column-major; the packed
    parameter vector is w = [vec A; vec B; vec C].
    In torch/numpy a column-major I×R matrix is the row-major array A_t of
    shape (R, I) (A_t[r, i] = a_ir); `pack_w` / `unpack_w` convert.

Workload recipes (BASELINE.json `configs`, readings in DESIGN.md §3):
  c1 20³ R=3     N(0,1) factors, T = [[A,B,C]] + 1e-3·N(0,1); points w*, w* + sqrt(0.1)·N
  c2 200³ R=10   N(0,1) unit-column factors, SNR 40 dB; point = independent N(0,1)
  c3 500³ R=20   collinear factors 0.9·s + sqrt(0.19)·u_r, SNR 30 dB; points w* and N(0,1)
  c4 4000×800×400 R=50  U(0,1) factors, noise 0.1·N(0,1); point = independent U(0,1)
  c5 1200³ R=100 N(0,1) factors, noise std 1e-2·σ_T; point = independent N(0,1)

Randomness: every array is drawn from its own torch.Generator seeded by
(seed, array id[, slice index]); the noise of frontal slice k has its own
generator, so any K-range of T can be generated on its own (K-sharding) and is
bit-identical to the same slices of the full tensor generated on the same
device type.
"""
from __future__ import annotations

import hashlib
import math
from dataclasses import dataclass, field

import numpy as np
import torch


@dataclass(frozen=True)
class Config:
    name: str
    I: int
    J: int
    K: int
    R: int
    factors: str            # "normal", "normal_unit", "collinear", "uniform"
    noise: str              # "sigma", "snr_db", "sigma_T_frac"
    noise_value: float
    points: tuple = ("random",)
    lam: float = 1e-3
    cg_iters: int = 0
    desc: str = ""

    @property
    def n(self) -> int:
        return self.R * (self.I + self.J + self.K)

    @property
    def t_bytes(self) -> int:
        return 8 * self.I * self.J * self.K


CONFIGS = {
    "c1": Config("c1", 20, 20, 20, 3, "normal", "sigma", 1e-3, ("true", "perturbed"), 1e-3, 10,
                 "20x20x20 R=3, N(0,1) factors (seed 0), +N(0,1e-6) noise; points w* and w*+N(0,0.1)"),
    "c2": Config("c2", 200, 200, 200, 10, "normal_unit", "snr_db", 40.0, ("random",), 1e-3, 10,
                 "200^3 R=10, unit-column N(0,1) factors, SNR 40 dB; point random N(0,1)"),
    "c3": Config("c3", 500, 500, 500, 20, "collinear", "snr_db", 30.0, ("true", "random"), 1e-3, 10,
                 "500^3 R=20, collinearity 0.9, SNR 30 dB; 10 CG iterations, lambda=1e-3"),
    "c4": Config("c4", 4000, 800, 400, 50, "uniform", "sigma", 0.1, ("random_uniform",), 1e-3, 10,
                 "4000x800x400 R=50, U(0,1) factors, +N(0,0.01) noise; point random U(0,1)"),
    "c5": Config("c5", 1200, 1200, 1200, 100, "normal", "sigma_T_frac", 1e-2, ("random",), 1e-3, 20,
                 "1200^3 R=100, N(0,1) factors, +N(0,1e-2*sigma_T) noise; f, grad, 20 CG matvecs"),
}


def _seed(*parts) -> int:
    h = hashlib.sha256(("/".join(str(p) for p in parts)).encode()).digest()
    return int.from_bytes(h[:8], "little") & ((1 << 63) - 1)


def _gen(device, *parts) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(_seed(*parts))
    return g


def randn(shape, device, *parts) -> torch.Tensor:
    return torch.randn(shape, generator=_gen(device, *parts), dtype=torch.float64, device=device)


def rand(shape, device, *parts) -> torch.Tensor:
    return torch.rand(shape, generator=_gen(device, *parts), dtype=torch.float64, device=device)


# ----------------------------------------------------------------------------- layout helpers
def pack_w(A_t: torch.Tensor, B_t: torch.Tensor, C_t: torch.Tensor) -> torch.Tensor:
    """w = [vec A; vec B; vec C] from row-major (R, I_l) arrays (= column-major I_l×R)."""
    return torch.cat([A_t.reshape(-1), B_t.reshape(-1), C_t.reshape(-1)]).contiguous()


def unpack_w(w, I: int, J: int, K: int, R: int):
    """Views (R,I), (R,J), (R,K) of a packed vector (torch or numpy)."""
    a, b = R * I, R * I + R * J
    return w[:a].reshape(R, I), w[a:b].reshape(R, J), w[b:b + R * K].reshape(R, K)


# ----------------------------------------------------------------------------- factor draws
def _factor(kind: str, R: int, n: int, device, *parts) -> torch.Tensor:
    if kind == "normal":
        return randn((R, n), device, *parts)
    if kind == "normal_unit":
        x = randn((R, n), device, *parts)
        return x / torch.linalg.vector_norm(x, dim=1, keepdim=True)
    if kind == "uniform":
        return rand((R, n), device, *parts)
    if kind == "collinear":
        # column r = 0.9 s + sqrt(0.19) u_r with s, u_r unit-normalised N(0,1) (BASELINE c3).
        s = randn((1, n), device, *parts, "shared")
        s = s / torch.linalg.vector_norm(s)
        u = randn((R, n), device, *parts, "indep")
        u = u / torch.linalg.vector_norm(u, dim=1, keepdim=True)
        return 0.9 * s + math.sqrt(0.19) * u
    raise ValueError(kind)


def _outer_BA(A_t, B_t) -> torch.Tensor:
    """(R, J*I) rows b_r ⊗ a_r (i fastest) — the clean slice k is sum_r c_kr (b_r ⊗ a_r)."""
    return (B_t[:, :, None] * A_t[:, None, :]).reshape(A_t.shape[0], -1)


def _clean_slab(BA, C_t, k0, k1, J, I) -> torch.Tensor:
    """Clean slices [[A,B,C]][:, :, k0:k1] as a (k1-k0, J, I) tensor (workload recipe)."""
    return (C_t[:, k0:k1].transpose(0, 1) @ BA).reshape(k1 - k0, J, I)


@dataclass
class Problem:
    cfg: Config
    T: torch.Tensor                 # (K_local, J, I) fp64, first-index-fastest T
    k_begin: int                    # first global slice held in T
    true: tuple                     # (A_t, B_t, C_t) true factors, row-major (R, I_l)
    points: dict = field(default_factory=dict)   # name -> packed w (full K)
    sigma: float = 0.0              # noise std actually used
    device: str = "cpu"

    def w(self, point: str) -> torch.Tensor:
        return self.points[point]


def make_problem(name: str, device="cpu", seed: int = 0, k_range=None, slab: int = 16,
                 dims=None, noise_value=None) -> Problem:
    """Build the seeded workload `name` on `device`.

    k_range=(k0, k1) keeps only slices k0..k1-1 of T (K-sharding); everything
    that depends on all of T (SNR / σ_T scaling) is still computed from every
    slice, so a shard is bit-identical to the same slices of the full tensor.
    dims=(I,J,K,R) overrides the shape (tests use the recipes at reduced size); noise_value overrides the
    recipe's noise level in its own unit (sigma, SNR in dB, or fraction of sigma_T) — the tests of the
    cancellation guard (reading R31) use c3's recipe at other SNRs.
    """
    cfg = CONFIGS[name]
    if dims is not None:
        I, J, K, R = dims
        cfg = Config(cfg.name, I, J, K, R, cfg.factors, cfg.noise, cfg.noise_value, cfg.points,
                     cfg.lam, cfg.cg_iters, cfg.desc + f" (reduced to {I}x{J}x{K} R={R})")
    if noise_value is not None:
        cfg = Config(cfg.name, cfg.I, cfg.J, cfg.K, cfg.R, cfg.factors, cfg.noise, float(noise_value), cfg.points,
                     cfg.lam, cfg.cg_iters, cfg.desc + f" (noise {cfg.noise} = {noise_value})")
    I, J, K, R = cfg.I, cfg.J, cfg.K, cfg.R
    k0, k1 = (0, K) if k_range is None else k_range
    dev = torch.device(device)
    A_t = _factor(cfg.factors, R, I, dev, seed, name, "A")
    B_t = _factor(cfg.factors, R, J, dev, seed, name, "B")
    C_t = _factor(cfg.factors, R, K, dev, seed, name, "C")

    # Pass 1: norms of the clean tensor and of the raw noise, slab by slab (all K).
    need_norms = cfg.noise in ("snr_db", "sigma_T_frac")
    clean_sq = 0.0
    noise_sq = 0.0
    BA = _outer_BA(A_t, B_t)
    if need_norms:
        for s0 in range(0, K, slab):
            s1 = min(K, s0 + slab)
            X = _clean_slab(BA, C_t, s0, s1, J, I)
            clean_sq += float(torch.sum(X * X))
            if cfg.noise == "snr_db":
                for k in range(s0, s1):
                    nk = randn((J, I), dev, seed, name, "noise", k)
                    noise_sq += float(torch.sum(nk * nk))
            del X
    if cfg.noise == "sigma":
        sigma = cfg.noise_value
    elif cfg.noise == "snr_db":
        # ||N|| = ||T_clean|| * 10^(-SNR/20) exactly (reading R10)
        sigma = math.sqrt(clean_sq) * 10.0 ** (-cfg.noise_value / 20.0) / math.sqrt(noise_sq)
    elif cfg.noise == "sigma_T_frac":
        sigma = cfg.noise_value * math.sqrt(clean_sq / (I * J * K))
    else:
        raise ValueError(cfg.noise)

    # Pass 2: the local slices.
    T = torch.empty((k1 - k0, J, I), dtype=torch.float64, device=dev)
    for s0 in range(k0, k1, slab):
        s1 = min(k1, s0 + slab)
        T[s0 - k0:s1 - k0] = _clean_slab(BA, C_t, s0, s1, J, I)
        for k in range(s0, s1):
            T[k - k0] += sigma * randn((J, I), dev, seed, name, "noise", k)

    del BA
    pts = {}
    for p in cfg.points:
        if p == "true":
            pts["true"] = pack_w(A_t, B_t, C_t)
        elif p == "perturbed":
            d = randn((cfg.n,), dev, seed, name, "perturb")
            pts["perturbed"] = pack_w(A_t, B_t, C_t) + math.sqrt(0.1) * d
        elif p == "random":
            pts["random"] = pack_w(randn((R, I), dev, seed, name, "x0A"), randn((R, J), dev, seed, name, "x0B"),
                                   randn((R, K), dev, seed, name, "x0C"))
        elif p == "random_uniform":
            pts["random_uniform"] = pack_w(rand((R, I), dev, seed, name, "x0A"), rand((R, J), dev, seed, name, "x0B"),
                                           rand((R, K), dev, seed, name, "x0C"))
    return Problem(cfg, T, k0, (A_t, B_t, C_t), pts, sigma, str(dev))


def random_vector(n: int, device="cpu", *parts) -> torch.Tensor:
    """A seeded N(0,1) vector of length n (matvec / CG right-hand sides in tests)."""
    return randn((n,), torch.device(device), "vec", *parts)


def shard_range(K: int, rank: int, world: int):
    """Contiguous, balanced K-range of `rank`: first K%world ranks get one extra slice."""
    base, extra = divmod(K, world)
    k0 = rank * base + min(rank, extra)
    return k0, k0 + base + (1 if rank < extra else 0)


def cg_budget(maxiter: int, seed: int = 0):
    """Tensor Fox's random CG budget: at dGN iteration k, cg_maxiter is a uniform random
    integer in [1 + ceil(k^0.4), 2 + ceil(k^0.9)]. These are the random numbers the method draws; they are
    drawn here (seeded) and passed to both the oracle and the CUDA path as an input."""
    rng = np.random.default_rng(_seed(seed, "cg_budget"))
    ks = np.arange(1, maxiter + 1)
    lo = 1 + np.ceil(ks ** 0.4).astype(np.int64)
    hi = 2 + np.ceil(ks ** 0.9).astype(np.int64)
    return rng.integers(lo, hi + 1).astype(np.int32)


def omega_blocks(dims, R: int, device="cpu", seed: int = 0, tag: str = "omega") -> torch.Tensor:
    """Start blocks of the randomized truncated SVD (rand_svd): for each mode l an
    I_l × P_l block of i.i.d. N(0,1) entries (column-major), P_l = min(I_l, R), concatenated
    [Ω1 | Ω2 | Ω3]. These are the random numbers the compression stage draws; they are drawn here
    (seeded) and passed to the CUDA path as an input."""
    dev = torch.device(device)
    parts = []
    for l, n in enumerate(dims):
        P = min(n, R)
        parts.append(randn((P, n), dev, seed, tag, l).reshape(-1))   # (P, n) row-major = n x P column-major
    return torch.cat(parts)
