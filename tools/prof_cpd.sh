ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cpd_launches.csv python - <<PY > /dev/null 2>&1
import sys, torch, math
sys.path.insert(0, ".")
import paper_2110_05997_b200 as tf, synth
P = synth.make_problem("c5", "cuda"); c = P.cfg
I, J, K, R = c.I, c.J, c.K, c.R
ctx = tf.Context(0); d = tf.Dims(I, J, K, R)
Om = synth.omega_blocks((I, J, K), R, "cuda")
cgi = synth.cg_budget(200, seed=0)
Ps = [min(x, R) for x in (I, J, K)]
w0 = torch.cat([synth.randn((R, p), torch.device("cuda"), "cpd-init", l).reshape(-1) for l, p in enumerate(Ps)])
W, lam, out, hist = ctx.tf_cpd(d, P.T, Om, cgi, w0_core=w0, maxiter=200, tol=1e-6, sequential=True)
print(out)
PY
python - <<PY
import csv, collections
lines=open("gpurun_out/cpd_launches.csv").read().splitlines()
i=[k for k,l in enumerate(lines) if l.startswith('"ID"')][0]
rows=[r for r in csv.DictReader(lines[i:]) if r.get("Metric Name")=="gpu__time_duration.sum"]
agg=collections.defaultdict(lambda:[0,0.0])
for r in rows:
    k=r["Kernel Name"].split("(")[0][:70]; agg[k][0]+=1; agg[k][1]+=float(r["Metric Value"].replace(",",""))/1e6
tot=sum(t for c,t in agg.values())
print("total", tot)
for k,(c,t) in sorted(agg.items(), key=lambda x:-x[1][1])[:25]: print(f"{c:6d} {t:9.3f} ms {100*t/tot:5.1f}%  {k}")
PY
