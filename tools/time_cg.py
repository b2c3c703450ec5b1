"""Device timing of tf_cg_solve / tf_gn_matvec on a config (development aid)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2110_05997_b200 as tf
import synth

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
cfg = synth.CONFIGS[name]
I, J, K, R = cfg.I, cfg.J, cfg.K, cfg.R
g = torch.Generator(device="cuda").manual_seed(1)
w = torch.randn(cfg.n, generator=g, dtype=torch.float64, device="cuda")
rhs = torch.randn(cfg.n, generator=g, dtype=torch.float64, device="cuda")
d = tf.Dims(I, J, K, R)
ctx = tf.Context(0)
grams = ctx.tf_grams(d, w)
x = torch.empty_like(w)
y = torch.empty_like(w)
for _ in range(3):
    ctx.tf_cg_solve(d, grams, w, rhs, cfg.lam, cfg.cg_iters or 10, 0.0, False, x)
    ctx.tf_gn_matvec(d, grams, w, rhs, cfg.lam, y)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = 10
e0.record()
for _ in range(n):
    ctx.tf_cg_solve(d, grams, w, rhs, cfg.lam, cfg.cg_iters or 10, 0.0, False, x)
e1.record(); torch.cuda.synchronize()
t_cg = e0.elapsed_time(e1) / n
e0.record()
for _ in range(n):
    ctx.tf_gn_matvec(d, grams, w, rhs, cfg.lam, y)
e1.record(); torch.cuda.synchronize()
t_mv = e0.elapsed_time(e1) / n
print(f"{name}: tf_cg_solve({cfg.cg_iters or 10}) {t_cg*1000:.1f} us ({t_cg*1000/(cfg.cg_iters or 10):.1f} us/iter), "
      f"tf_gn_matvec {t_mv*1000:.1f} us")
import ctypes, os
if os.environ.get("TF_CG_TSTAMP"):
    L = ctypes.CDLL(tf.LIB_PATH)
    ctx.tf_cg_solve(d, grams, w, rhs, cfg.lam, cfg.cg_iters or 10, 0.0, False, x)
    L.tf_cg_debug_dump()
