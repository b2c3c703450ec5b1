"""Device timing of the compression stage (NEXT #3) on a config: unfolding Grams per mode, eigenpairs,
core, and the whole tf_compress (development aid; CUDA events on the ctx stream)."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2110_05997_b200 as tf
import synth

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
t0 = time.time()
P = synth.make_problem(name, "cuda")
torch.cuda.synchronize()
c = P.cfg
I, J, K, R = c.I, c.J, c.K, c.R
print(f"{name}: generated in {time.time()-t0:.1f}s", flush=True)
d = tf.Dims(I, J, K, R)
ctx = tf.Context(0)
st = ctx.stream


def timed(fn, n=reps):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(n):
        out = fn()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n, out


dims = (I, J, K)
for mode in (1, 2, 3):
    ms, _ = timed(lambda: ctx.tf_unfolding_grams(d, P.T, modes=(mode,)))
    n = dims[mode - 1]
    # G = X X^T with X = T_(l) (n x IJK/n): full product 2 n IJK flops; symmetric (algorithmic) (n+1) IJK
    flops_full = 2.0 * n * I * J * K
    flops_sym = 1.0 * (n + 1) * I * J * K
    print(f"{name}: gram mode {mode}: {ms:.2f} ms  {flops_sym/ms/1e9:.2f} TF/s (symmetric, algorithmic) "
          f"{flops_full/ms/1e9:.2f} TF/s (full-product equivalent)", flush=True)
Om = synth.omega_blocks(dims, R, "cuda")
G = ctx.tf_unfolding_grams(d, P.T, modes=(1,))[0]
Pm = min(I, R)
ms, (U, lam, it) = timed(lambda: ctx.tf_sym_eig_top(I, G, Pm, Om[:I * Pm]), 1)
print(f"{name}: eig mode 1 (n={I}, P={Pm}): {ms:.2f} ms, {it} iterations", flush=True)
Ps = [min(n, R) for n in dims]
U1 = torch.linalg.qr(torch.randn(I, Ps[0], dtype=torch.float64, device="cuda"))[0].T.contiguous().reshape(-1)
U2 = torch.linalg.qr(torch.randn(J, Ps[1], dtype=torch.float64, device="cuda"))[0].T.contiguous().reshape(-1)
U3 = torch.linalg.qr(torch.randn(K, Ps[2], dtype=torch.float64, device="cuda"))[0].T.contiguous().reshape(-1)
ms, _ = timed(lambda: ctx.tf_multilinear_core(d, P.T, U1, Ps[0], U2, Ps[1], U3, Ps[2]))
fl = 2.0 * Ps[0] * I * J * K + 2.0 * Ps[0] * Ps[1] * J * K + 2.0 * Ps[0] * Ps[1] * Ps[2] * K
print(f"{name}: core ({Ps}): {ms:.2f} ms  {fl/ms/1e9:.2f} TF/s", flush=True)
t0 = time.time()
ms, out = timed(lambda: ctx.tf_compress(d, P.T, Om, mlsvd_tol=1e-6), 1)
print(f"{name}: tf_compress: {ms:.1f} ms (wall {1e3*(time.time()-t0):.0f} ms incl. warm-up), ranks {out['ranks']}, "
      f"eig iterations {out['eig_iters']}", flush=True)
