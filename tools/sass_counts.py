"""Per-kernel SASS instruction counts of the built library (cuobjdump -sass, run here on the host): the Blackwell
path evidence — DMMA (FP64 tensor core), UTMALDG/UBLKCP (TMA tensor / bulk copies), LDTM/STTM (tensor memory),
LDGSTS (cp.async), SYNCS (mbarrier), BAR (block barriers). Static counts per kernel, not executed counts."""
import collections
import json
import re
import subprocess
import sys

so = sys.argv[1] if len(sys.argv) > 1 else "paper_2110_05997_b200/libtf.so"
sass = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
pat = {"DMMA": r"\bDMMA\b", "DFMA": r"\bDFMA\b", "UTMALDG": r"\bUTMALDG\b", "UBLKCP": r"\bUBLKCP\b",
       "LDTM": r"\bLDTM\b", "STTM": r"\bSTTM\b", "UTCATOMSWS/ALLOC": r"\bUTC\w*\b", "LDGSTS": r"\bLDGSTS\b",
       "SYNCS": r"\bSYNCS\b", "BAR": r"\bBAR\b", "WARPSYNC": r"\bWARPSYNC\b"}
out = collections.OrderedDict()
cur = None
for line in sass.splitlines():
    m = re.match(r"\s*Function : (\S+)", line)
    if m:
        cur = m.group(1)
        out[cur] = collections.Counter()
        continue
    if cur and "/*" in line:
        for k, p in pat.items():
            if re.search(p, line):
                out[cur][k] += 1


def short(n):
    n = n.replace("_ZN3tfk", "")
    return n[:90]


res = {short(k): dict(v) for k, v in out.items() if v.get("DMMA") or v.get("UTMALDG") or v.get("LDTM") or
       v.get("LDGSTS")}
print(json.dumps({"library": so, "note": __doc__.replace("\n", " "), "kernels": res}, indent=1))
