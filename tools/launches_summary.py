"""Summarise an ncu --metrics gpu__time_duration.sum launch list (csv) into per-kernel totals and shares."""
import csv
import json
import sys

src, cmd = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
note = sys.argv[3] if len(sys.argv) > 3 else ""
rows = [r for r in csv.DictReader(l for l in open(src) if l.startswith('"'))]
k = {}
for r in rows:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = r["Kernel Name"].split("(")[0]
    scale = {"ns": 1e-6, "us": 1e-3, "ms": 1.0}[r["Metric Unit"]]
    e = k.setdefault(name, {"launches": 0, "total_ms": 0.0})
    e["launches"] += 1
    e["total_ms"] += float(r["Metric Value"].replace(",", "")) * scale
tot = sum(e["total_ms"] for e in k.values())
for e in k.values():
    e["total_ms"] = round(e["total_ms"], 4)
    e["share"] = round(e["total_ms"] / tot, 4)
out = {"command": cmd, "note": note,
       "kernels": dict(sorted(k.items(), key=lambda kv: -kv[1]["total_ms"])), "total_ms": round(tot, 4)}
print(json.dumps(out, indent=1))
