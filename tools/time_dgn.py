"""Per-iteration time of the dGN loop (tf_cpd_dgn) on an exact-rank-plus-noise cube (development aid)."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2110_05997_b200 as tf
import synth

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100
R = int(sys.argv[2]) if len(sys.argv) > 2 else 100
its = int(sys.argv[3]) if len(sys.argv) > 3 else 30
A, B, C = (synth.randn((R, n), torch.device("cuda"), "dgn-t", l) for l in range(3))
T = torch.einsum("ri,rj,rk->kji", A, B, C).contiguous() + 1e-2 * synth.randn((n, n, n), torch.device("cuda"), "dgn-n")
w0 = synth.randn((3 * n * R,), torch.device("cuda"), "dgn-w0")
ctx = tf.Context(0)
d = tf.Dims(n, n, n, R)
cgi = [10] * its
w = w0.clone()
ctx.tf_cpd_dgn(d, T, w, cgi, maxiter=3, tol=0.0)
torch.cuda.synchronize()
w = w0.clone()
t0 = time.perf_counter()
out, hist = ctx.tf_cpd_dgn(d, T, w, cgi, maxiter=its, tol=0.0)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
print(f"dgn {n}^3 R={R}: {its} iterations (10 CG each) in {dt*1e3:.1f} ms = {dt*1e3/its:.3f} ms/iteration; "
      f"rel_err {out['rel_err']:.3e}", flush=True)
