"""One rank's K-sharded c5 step at N GPUs (tf_cpd_eval on the K/N shard, returning the full-factor Grams, + tf_cg_solve), timed with
CUDA events; run under `ncu --metrics gpu__time_duration.sum` for the per-kernel split (development aid)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2110_05997_b200 as tf
import synth

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
N = int(sys.argv[2]) if len(sys.argv) > 2 else 8
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
cfg = synth.CONFIGS[name]
I, J, K, R = cfg.I, cfg.J, cfg.K, cfg.R
P = synth.make_problem(name, "cuda")
w = P.w(cfg.points[-1])
ctx = tf.Context(0)
grams = torch.empty(3 * R * R, dtype=torch.float64, device="cuda")
x = torch.empty(cfg.n, dtype=torch.float64, device="cuda")
k1 = (K + N - 1) // N
d = tf.Dims(I, J, k1, R, K_total=K, k_begin=0)
dg = tf.Dims(I, J, K, R)
Tl = P.T[:k1]
f = torch.empty(1, dtype=torch.float64, device="cuda")
g = torch.empty(cfg.n, dtype=torch.float64, device="cuda")


def step():
    ctx.tf_cpd_eval(d, Tl, w, f, g, grams)
    ctx.tf_cg_solve(dg, grams, w, -g, cfg.lam, cfg.cg_iters or 10, 0.0, False, x)


for _ in range(2):
    step()
torch.cuda.synchronize()
e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
tot_eval = tot_cg = 0.0
for _ in range(reps):
    e[0].record()
    ctx.tf_cpd_eval(d, Tl, w, f, g, grams)
    e[1].record()
    ctx.tf_cg_solve(dg, grams, w, -g, cfg.lam, cfg.cg_iters or 10, 0.0, False, x)
    e[2].record()
    torch.cuda.synchronize()
    tot_eval += e[0].elapsed_time(e[1])
    tot_cg += e[1].elapsed_time(e[2])
print(f"{name} N={N} shard {k1} slices: eval {tot_eval/reps:.3f} ms, cg {tot_cg/reps:.3f} ms, "
      f"step {(tot_eval+tot_cg)/reps:.3f} ms")
