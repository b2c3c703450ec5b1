"""One pass over every kernel family at small sizes, for compute-sanitizer (memcheck / racecheck / synccheck).

c1 (20^3, R=3) and c2 (200^3, R=10) in both evaluation forms, a reduced c3 shape (130x70x40, R=20) in the forced
Pi form (the TMEM / TMA / mbarrier path), the GN matvec and CG through the row-owned, grid and one-CTA kernels,
a short dGN loop, ST-MLSVD compression and one CP-ALS sweep. Prints one line per step; exits non-zero on error.
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2110_05997_b200 as tf  # noqa: E402
import synth  # noqa: E402

ctx = tf.Context(0)
cases = [("c1", None, "perturbed"), ("c2", None, "random"), ("c3", (130, 70, 40, 20), "random")]
if len(sys.argv) > 1 and sys.argv[1] == "small":      # racecheck: shared-memory hazard tracking is slow
    cases = [("c1", None, "perturbed"), ("c3", (70, 66, 20, 20), "random")]
for name, dims, point in cases:
    P = synth.make_problem(name, "cpu", dims=dims)
    c = P.cfg
    d = tf.Dims(c.I, c.J, c.K, c.R)
    T = P.T.cuda().contiguous()
    w = P.w(point).cuda().contiguous()
    for form in ("residual", "pi"):
        ctx.set_eval_form(form)
        f, g = ctx.tf_cpd_eval(d, T, w)
        torch.cuda.synchronize()
        print(f"{name} eval {form}: f={f.item():.6e} fell_back={ctx.eval_fell_back()}", flush=True)
    ctx.set_eval_form("auto")
    grams = ctx.tf_grams(d, w)
    y = ctx.tf_gn_matvec(d, grams, w, g, 1e-3)
    for kern in ("auto", "grid"):
        if kern == "grid":
            os.environ["TF_CG_KERNEL"] = "grid"
        for grid in (0, 7):
            ctx.set_cg_grid(grid)
            x, it, r2 = ctx.tf_cg_solve(d, grams, w, -g, 1e-3, 5, 0.0, True)
            torch.cuda.synchronize()
            print(f"{name} cg kernel={kern} grid={grid}: iters={it} r2={r2:.3e}", flush=True)
        os.environ.pop("TF_CG_KERNEL", None)
    ctx.set_cg_grid(0)
    wd = w.clone()
    out, _ = ctx.tf_cpd_dgn(d, T, wd, synth.cg_budget(3, seed=0), maxiter=3, tol=0.0)
    print(f"{name} dgn: {out}", flush=True)
    Om = synth.omega_blocks((c.I, c.J, c.K), c.R, "cuda")
    comp = ctx.tf_compress(d, T, Om, mlsvd_tol=1e-6, sequential=True)
    print(f"{name} compress: ranks={comp['ranks']}", flush=True)
    wa = w.clone()
    ctx.tf_als(d, T, wa, 1)
    torch.cuda.synchronize()
    print(f"{name} als: ok", flush=True)
ctx.close()
print("sanitize_run: done")
