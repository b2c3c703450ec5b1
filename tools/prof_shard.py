"""Warm per-kernel device times of one rank's K-sharded c5 step (torch.profiler / CUPTI), development aid."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2110_05997_b200 as tf
import synth

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
N = int(sys.argv[2]) if len(sys.argv) > 2 else 8
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
f = torch.empty(1, dtype=torch.float64, device="cuda")
g = torch.empty(cfg.n, dtype=torch.float64, device="cuda")


def step():
    ctx.tf_cpd_eval(d, P.T[:k1], w, f, g, grams)
    ctx.tf_cg_solve(dg, grams, w, -g, cfg.lam, cfg.cg_iters or 10, 0.0, False, x)


for _ in range(3):
    step()
torch.cuda.synchronize()
reps = 5
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    for _ in range(reps):
        step()
    torch.cuda.synchronize()
tot = {}
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        k = e.name.split("(")[0][:60]
        tot.setdefault(k, [0, 0.0])
        tot[k][0] += 1
        tot[k][1] += e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
s = 0.0
for k, (n_, us) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
    s += us / reps
    print(f"{k:60s} {n_ // reps:3d}/step {us / reps:9.1f} us/step")
print(f"total {s:.1f} us/step")
