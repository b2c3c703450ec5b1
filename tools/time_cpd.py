"""The whole Tensor Fox flow (tf_cpd) on a config: energy vs random initialisation (development aid)."""
import math
import sys

import torch

sys.path.insert(0, ".")
import paper_2110_05997_b200 as tf
import synth

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
maxiter = int(sys.argv[2]) if len(sys.argv) > 2 else 200
P = synth.make_problem(name, "cuda")
c = P.cfg
I, J, K, R = c.I, c.J, c.K, c.R
d = tf.Dims(I, J, K, R)
ctx = tf.Context(0)
Om = synth.omega_blocks((I, J, K), R, "cuda")
cgi = synth.cg_budget(maxiter, seed=0)
noise = P.sigma * math.sqrt(I * J * K) / math.sqrt(float(torch.sum(P.T * P.T)))
Ps = [min(n, R) for n in (I, J, K)]
w0 = torch.cat([synth.randn((R, p), torch.device("cuda"), "cpd-init", l).reshape(-1) for l, p in enumerate(Ps)])
for label, kw in (("energy", {}), ("random", {"w0_core": w0})):
    for seq in (True, False):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(ctx.stream)
        W, lam, out, hist = ctx.tf_cpd(d, P.T, Om, cgi, maxiter=maxiter, tol=1e-6, sequential=seq, **kw)
        e1.record(ctx.stream)
        torch.cuda.synchronize()
        print(f"{name} init={label} st={seq}: {e0.elapsed_time(e1):.0f} ms, ranks {out['ranks']}, dGN {out['dgn']['iters']} "
              f"it (stop {out['dgn']['reason']}), rel_err {out['rel_err']:.4e} (noise {noise:.2e})", flush=True)
