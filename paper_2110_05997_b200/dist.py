"""K-sharded multi-GPU evaluation: one process per GPU, frontal slices split
into contiguous balanced ranges, one SUM all-reduce of the packed [grad | f] buffer.

Each rank evaluates its slices T[:, :, k0:k1] with the replicated factors w (tf_cpd_eval with
K_total / k_begin): dF/dA, dF/dB and f are partial sums, dF/dC holds only its own rows (zeros
elsewhere), so a single elementwise SUM all-reduce over NVLink (NCCL through torch.distributed,
on the evaluation stream) gives every rank the full f and gradient. The Gauss-Newton matvec and
CG are O(R^2 sum I) and run replicated (no communication).

The host-side logic (partition, packing, reduction) is independent of the evaluator so that it
can be exercised on CPU with the gloo backend (tests/test_dist_gloo.py); the product path always
passes the CUDA evaluator.
"""
from __future__ import annotations

from typing import Callable

import torch
import torch.distributed as dist


def shard_range(K: int, rank: int, world: int):
    """Contiguous balanced K-range: the first K % world ranks get one extra slice."""
    base, extra = divmod(K, world)
    k0 = rank * base + min(rank, extra)
    return k0, k0 + base + (1 if rank < extra else 0)


class ShardedEvaluator:
    """Evaluate (f, grad) of the full problem from this rank's slices.

    eval_fn(dims, T_local, w, f_out, grad_out) must write the local partials; by default it is
    the CUDA path `Context.tf_cpd_eval`.
    """

    def __init__(self, I: int, J: int, K: int, R: int, rank: int | None = None, world: int | None = None,
                 ctx=None, eval_fn: Callable | None = None, group=None, device=None):
        self.I, self.J, self.K, self.R = I, J, K, R
        self.group = group
        if world is None:
            world = dist.get_world_size(group) if dist.is_initialized() else 1
        if rank is None:
            rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.rank, self.world = rank, world
        self.k0, self.k1 = shard_range(K, rank, world)
        self.n = R * (I + J + K)
        if eval_fn is None:
            if ctx is None:
                raise ValueError("need a Context (CUDA path) or an explicit eval_fn")
            from . import Dims

            def eval_fn(d, T, w, f, g, grams=None):
                ctx.tf_cpd_eval(d, T, w, f, g, grams)
            self._Dims = Dims
        else:
            from types import SimpleNamespace
            self._Dims = lambda **kw: SimpleNamespace(**kw)
        self.eval_fn = eval_fn
        self.ctx = ctx
        self.device = device
        self.buf = None

    @property
    def local_dims(self):
        return self._Dims(I=self.I, J=self.J, K=self.k1 - self.k0, R=self.R, ldT=0, K_total=self.K,
                          k_begin=self.k0)

    def packed(self, device):
        if self.buf is None or self.buf.device != torch.device(device):
            self.buf = torch.empty(self.n + 1, dtype=torch.float64, device=device)
        return self.buf

    def __call__(self, T_local: torch.Tensor, w: torch.Tensor, allreduce: bool = True, grams=None):
        """Returns views (f[1], grad[n]) of the packed buffer, globally reduced when allreduce=True. With
        `grams` (3R^2, device) the CUDA evaluator also returns the Grams of the full (replicated) factors."""
        buf = self.packed(w.device)
        grad, f = buf[:self.n], buf[self.n:]
        if grams is not None:
            self.eval_fn(self.local_dims, T_local, w, f, grad, grams)
        else:
            self.eval_fn(self.local_dims, T_local, w, f, grad)
        if allreduce and self.world > 1:
            stream = getattr(self.ctx, "stream", None) if buf.is_cuda else None
            if stream is not None:
                # the evaluation was enqueued on the library's stream; NCCL orders after torch's current stream,
                # so run the collective on the evaluation stream itself (no read of buf before the kernels end)
                with torch.cuda.stream(stream):
                    dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=self.group)
            else:
                dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=self.group)
        return f, grad


def allreduce_hook(group=None):
    """The SUM all-reduce a K-sharded tf_cpd_dgn_sharded call needs (NCCL over NVLink on GPUs; any
    torch.distributed backend): replaces `buf` in place by its elementwise sum over the ranks of `group`."""
    def hook(buf: torch.Tensor):
        if dist.is_initialized() and dist.get_world_size(group) > 1:
            dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)
    return hook


def sharded_dgn(ctx, I: int, J: int, K: int, R: int, T_local: torch.Tensor, w: torch.Tensor, cg_iters,
                rank: int | None = None, world: int | None = None, group=None, **kw):
    """Tensor Fox's dGN loop over K-sharded ranks: this rank holds T[:, :, k0:k1] (shard_range) and the full
    replicated w; returns what Context.tf_cpd_dgn_sharded returns (identical w on every rank)."""
    from . import Dims
    if world is None:
        world = dist.get_world_size(group) if dist.is_initialized() else 1
    if rank is None:
        rank = dist.get_rank(group) if dist.is_initialized() else 0
    k0, k1 = shard_range(K, rank, world)
    d = Dims(I, J, k1 - k0, R, K_total=K, k_begin=k0)
    return ctx.tf_cpd_dgn_sharded(d, T_local, w, cg_iters, allreduce_hook(group), **kw)


def sharded_cpd(ctx, I: int, J: int, K: int, R: int, T_local: torch.Tensor, Omega: torch.Tensor, cg_iters,
                rank: int | None = None, world: int | None = None, group=None, **kw):
    """The whole Tensor Fox flow over K-sharded ranks (ST-MLSVD compression with the Grams and the mode-3
    intermediate all-reduced, then the dGN on the core and the uncompression replicated): returns what
    Context.tf_cpd_sharded returns, identical on every rank."""
    from . import Dims
    if world is None:
        world = dist.get_world_size(group) if dist.is_initialized() else 1
    if rank is None:
        rank = dist.get_rank(group) if dist.is_initialized() else 0
    k0, k1 = shard_range(K, rank, world)
    d = Dims(I, J, k1 - k0, R, K_total=K, k_begin=k0)
    return ctx.tf_cpd_sharded(d, T_local, Omega, cg_iters, allreduce_hook(group), **kw)
