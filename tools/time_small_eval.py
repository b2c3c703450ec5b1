"""Device timing of tf_cpd_eval on small cubes (the compressed cores of the Tensor Fox flow)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2110_05997_b200 as tf
import synth

for n, R in ((100, 100), (60, 50), (20, 20), (100, 10)):
    T = synth.randn((n, n, n), torch.device("cuda"), "small-eval", n)
    w = synth.randn((3 * n * R,), torch.device("cuda"), "small-w", n, R)
    d = tf.Dims(n, n, n, R)
    ctx = tf.Context(0)
    for form in ("residual", "pi"):
        ctx.set_eval_form(form)
        f, g = ctx.tf_cpd_eval(d, T, w)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(ctx.stream)
        for _ in range(20):
            ctx.tf_cpd_eval(d, T, w, f, g)
        e1.record(ctx.stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 20
        print(f"{n}^3 R={R} {form}: {ms*1000:.1f} us/eval  {6*n**3*R/ms/1e9:.2f} TF/s (6IJKR)", flush=True)
    ctx.close()
