"""Device timing of the Pi-form evaluation on a c3-recipe tensor of given I J K R (development aid)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2110_05997_b200 as tf
import synth

I, J, K, R = (int(x) for x in sys.argv[1:5])
iters = int(sys.argv[5]) if len(sys.argv) > 5 else 20
P = synth.make_problem("c3", "cuda", dims=(I, J, K, R))
d = tf.Dims(I, J, K, R)
ctx = tf.Context(0)
ctx.set_eval_form("pi")
w = P.w("random")
f, g = ctx.tf_cpd_eval(d, P.T, w)
torch.cuda.synchronize()
ctx.set_timing(True)
ctx.kernel_stats(reset=True)
for _ in range(iters):
    ctx.tf_cpd_eval(d, P.T, w, f, g)
torch.cuda.synchronize()
kms, n, tot = ctx.kernel_stats()
fl = 4.0 * I * J * K * R
print(f"{I}x{J}x{K} R={R}: fused kernel {kms/n:.4f} ms, {fl/(kms/n*1e-3)/1e12:.2f} TFLOP/s (4IJKR), "
      f"frac {fl/(kms/n*1e-3)/37.14e12:.3f}", flush=True)
