"""Device timing of the CP-ALS path (NEXT #4): the three MTTKRPs and one ALS sweep on a config."""
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
w = P.w(c.points[-1]).clone()
st = ctx.stream
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for mode in (1, 2, 3):
    M = ctx.tf_mttkrp(d, P.T, w, mode)
    torch.cuda.synchronize()
    e0.record(st)
    ctx.tf_mttkrp(d, P.T, w, mode, M)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"{name}: mttkrp mode {mode}: {ms:.2f} ms  {2.0*I*J*K*R/ms/1e9:.2f} TF/s  "
          f"{8.0*I*J*K/ms/1e6:.0f} GB/s of T", flush=True)
ctx.tf_als(d, P.T, w, 1)
torch.cuda.synchronize()
e0.record(st)
ctx.tf_als(d, P.T, w, 1)
e1.record(st)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
print(f"{name}: ALS sweep: {ms:.2f} ms  ({6.0*I*J*K*R/ms/1e9:.2f} TF/s of MTTKRP flops)", flush=True)
