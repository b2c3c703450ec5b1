"""Quick device timing of tf_cpd_eval on a config (development aid)."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2110_05997_b200 as tf
import synth

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 5
t0 = time.time()
P = synth.make_problem(name, "cuda")
torch.cuda.synchronize()
c = P.cfg
print(f"{name}: generated in {time.time()-t0:.1f}s", flush=True)
d = tf.Dims(c.I, c.J, c.K, c.R)
ctx = tf.Context(0)
if len(sys.argv) > 3:
    ctx.set_eval_form(sys.argv[3])   # auto | residual | pi
w = P.w(P.cfg.points[-1])
f, g = ctx.tf_cpd_eval(d, P.T, w)
torch.cuda.synchronize()
ctx.set_timing(True)
ctx.kernel_stats(reset=True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(iters):
    ctx.tf_cpd_eval(d, P.T, w, f, g)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / iters
kms, n, tot = ctx.kernel_stats()
fb = ctx.eval_fell_back()
form = "residual" if fb != 0 else "pi"
flops = (6.0 if form == "residual" else 4.0) * c.I * c.J * c.K * c.R
print(f"{name}: eval {ms:.3f} ms/eval ({form} form), fused kernel {kms/n:.3f} ms, {flops/(kms/n*1e-3)/1e12:.2f} "
      f"TFLOP/s ({'6' if form == 'residual' else '4'}IJKR), {8*c.I*c.J*c.K/(kms/n*1e-3)/1e9:.0f} GB/s of T", flush=True)
