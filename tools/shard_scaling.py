"""Single-GPU projection of the K-sharded step: for N = 1, 2, 4, 8 time, on one B200, exactly the
work one rank of an N-GPU run does per step — tf_cpd_eval on its K/N-slice shard (k_begin = 0, K_total = K),
with the Grams of the full factors, and the replicated tf_cg_solve — and report t(1)/t(N). The NCCL all-reduce of [grad | f]
(R(I+J+K)+1 doubles, 2.9 MB at c5) cannot be measured on this single-GPU pool: the projection adds an explicit
allowance of ALLREDUCE_MS per step for N > 1 (an estimate, stated in the output: a ring all-reduce of 2.9 MB over
NVLink 5 moves 2 (N-1)/N x 2.9 MB per GPU, ~10 us at ~500 GB/s, plus ~20-40 us of NCCL launch/latency). This is a
projection from per-rank work, not a multi-GPU measurement."""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2110_05997_b200 as tf
import synth

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
ALLREDUCE_MS = float(sys.argv[2]) if len(sys.argv) > 2 else 0.05
cfg = synth.CONFIGS[name]
I, J, K, R = cfg.I, cfg.J, cfg.K, cfg.R
P = synth.make_problem(name, "cuda")
w = P.w(cfg.points[-1])
ctx = tf.Context(0)
n = cfg.n
grams = torch.empty(3 * R * R, dtype=torch.float64, device="cuda")
x = torch.empty(n, dtype=torch.float64, device="cuda")
dglob = tf.Dims(I, J, K, R)
out = {"config": name, "note": __doc__.replace("\n", " "), "allreduce_allowance_ms": ALLREDUCE_MS,
       "allreduce_allowance_source": "estimate (no multi-GPU box in this pool), not a measurement", "ranks": {}}
base = None
for N in (1, 2, 4, 8):
    k1 = (K + N - 1) // N   # the largest shard (rank 0 of the balanced split)
    d = tf.Dims(I, J, k1, R, K_total=K, k_begin=0)
    Tl = P.T[:k1]

    def step():
        f, g = ctx.tf_cpd_eval(d, Tl, w, grams=grams)
        if cfg.cg_iters:
            ctx.tf_cg_solve(dglob, grams, w, -g, cfg.lam, cfg.cg_iters, 0.0, False, x)

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    reps = 10
    for _ in range(reps):
        step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    base = base or ms
    tot = ms + (ALLREDUCE_MS if N > 1 else 0.0)
    out["ranks"][N] = {"shard_slices": k1, "ms_per_step_compute": ms,
                       "allreduce_allowance_ms": ALLREDUCE_MS if N > 1 else 0.0, "ms_per_step": tot,
                       "projected_speedup": base / tot, "projected_efficiency": base / tot / N}
    print(f"{name} N={N}: shard {k1} slices, {ms:.3f} ms per rank step (+{tot - ms:.3f} ms all-reduce allowance), "
          f"projected speedup {base/tot:.2f}x", flush=True)
print(json.dumps(out))
