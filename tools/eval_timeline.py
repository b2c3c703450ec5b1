"""Per-warp phase timeline of the fused kernel (needs libtf_prof.so built with -DTF_EVAL_PROFILE)."""
import ctypes, os, sys
os.environ["TF_LIB_PATH"] = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_2110_05997_b200", "libtf_prof.so")
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch
import paper_2110_05997_b200 as tf
import synth
name = sys.argv[1] if len(sys.argv) > 1 else "c5"
P = synth.make_problem(name, "cuda")
c = P.cfg
ctx = tf.Context(0)
d = tf.Dims(c.I, c.J, c.K, c.R)
w = P.w(c.points[-1])
for _ in range(2):
    ctx.tf_cpd_eval(d, P.T, w)
torch.cuda.synchronize()
ctypes.CDLL(tf.LIB_PATH).tf_eval_timeline_dump()
lib = ctypes.CDLL(tf.LIB_PATH)
lib.tf_eval_cta_dump(int(sys.argv[2]) if len(sys.argv) > 2 else 4096)
