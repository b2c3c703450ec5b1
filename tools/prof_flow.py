"""Warm per-kernel device times of the whole tf_cpd flow at c5 (torch.profiler / CUPTI), development aid."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2110_05997_b200 as tf
import synth

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
P = synth.make_problem(name, "cuda")
c = P.cfg
I, J, K, R = c.I, c.J, c.K, c.R
d = tf.Dims(I, J, K, R)
ctx = tf.Context(0)
Om = synth.omega_blocks((I, J, K), R, "cuda")
cgi = synth.cg_budget(200, seed=0)
Ps = [min(n, R) for n in (I, J, K)]
w0 = torch.cat([synth.randn((R, p), torch.device("cuda"), "cpd-init", l).reshape(-1) for l, p in enumerate(Ps)])
ctx.tf_cpd(d, P.T, Om, cgi, w0_core=w0, maxiter=200, tol=1e-6, sequential=True)
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA, torch.profiler.ProfilerActivity.CPU]) as prof:
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    W, lam, out, hist = ctx.tf_cpd(d, P.T, Om, cgi, w0_core=w0, maxiter=200, tol=1e-6, sequential=True)
    e1.record()
    torch.cuda.synchronize()
print(f"flow {e0.elapsed_time(e1):.1f} ms, dGN iters {out['dgn']['iters']}")
tot = {}
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        k = e.name.split("(")[0][:60]
        tot.setdefault(k, [0, 0.0])
        tot[k][0] += 1
        tot[k][1] += e.device_time_total
s = 0.0
for k, (n_, us) in sorted(tot.items(), key=lambda kv: -kv[1][1])[:25]:
    s += us
    print(f"{k:60s} {n_:5d} {us / 1000:9.2f} ms")
print(f"device total (top 25) {s / 1000:.1f} ms")
