"""Device timing of tf_sym_eig_top on a synthetic spectrum (development aid): n, P from argv."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2110_05997_b200 as tf
import synth

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1200
P = int(sys.argv[2]) if len(sys.argv) > 2 else 100
X = synth.randn((n, n + 40), torch.device("cuda"), "time-eig", n)
X[:, :P] *= torch.linspace(40, 5, P, dtype=torch.float64, device="cuda")
G = (X @ X.T).T.contiguous().reshape(-1)
Om = synth.randn((P, n), torch.device("cuda"), "time-eig-om", n).reshape(-1)
ctx = tf.Context(0)
ctx.tf_sym_eig_top(n, G, P, Om)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(ctx.stream)
U, lam, it = ctx.tf_sym_eig_top(n, G, P, Om)
e1.record(ctx.stream)
torch.cuda.synchronize()
print(f"eig n={n} P={P}: {e0.elapsed_time(e1):.2f} ms, {it} iterations", flush=True)
