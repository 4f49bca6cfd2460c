"""Stall samples by opcode and the top instructions of one kernel in an ncu
report (--set full --import-source on).  python tools/stall_report.py REP [N]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True,
                     text=True).stdout
kidx = int(sys.argv[3]) if len(sys.argv) > 3 else 0
blk = txt.split('"Kernel Name"')[1 + kidx]
rows = list(csv.reader(io.StringIO('"Kernel Name"' + blk)))
h = rows[1]
data = [r for r in rows[2:] if len(r) == len(h)]
ia, isrc = h.index("Address"), h.index("Source")
iw = h.index("Warp Stall Sampling (All Samples)")
sc = [(i, x) for i, x in enumerate(h) if x.startswith("stall_") and "Not Issued" not in x]
tot = sum(float(r[iw] or 0) for r in data)
op = defaultdict(float)
reason = defaultdict(float)
for r in data:
    toks = r[isrc].split()
    o = toks[1] if toks and toks[0].startswith("@") else (toks[0] if toks else "?")
    op[o.split(".")[0]] += float(r[iw] or 0)
    for i, x in sc:
        reason[x] += float(r[i] or 0)
rt = sum(reason.values())
print("by reason:", ", ".join(f"{k[6:]} {v / rt * 100:.1f}%" for k, v in
                              sorted(reason.items(), key=lambda kv: -kv[1])[:10]))
print("by opcode:", ", ".join(f"{k} {v / tot * 100:.1f}%" for k, v in
                              sorted(op.items(), key=lambda kv: -kv[1])[:12]))
for r in sorted(data, key=lambda r: -float(r[iw] or 0))[:n]:
    rs = sorted([(float(r[i] or 0), x[6:]) for i, x in sc], reverse=True)[:2]
    print(f"{float(r[iw]) / tot * 100:5.1f}% {r[ia][-5:]} {r[isrc][:58]:58s} "
          + " ".join(f"{x}:{v:.0f}" for v, x in rs))
