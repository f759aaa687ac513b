"""Top SASS lines of an ncu report by warp-stall samples, with the dominant
stall reasons, per kernel:  python scripts/ncu_source_top.py <report.ncu-rep> [n]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO("\n".join(l for l in txt.splitlines() if l.startswith('"')))))
sections, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "h": None, "data": []}
        sections.append(cur)
    elif cur is not None and cur["h"] is None:
        cur["h"] = r
    elif cur is not None:
        cur["data"].append(r)
for sec in sections:
    h, data = sec["h"], sec["data"]
    iS, iW = h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
    reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
    data = [r for r in data if r[iW].isdigit()]
    tot = sum(int(r[iW]) for r in data) or 1
    agg = {c: sum(int(r[h.index(c)] or 0) for r in data) for c in reasons}
    print(f"== {sec['name'][:90]}: samples {tot}, instructions {len(data)}")
    print("   by reason:", {k[6:]: round(v / tot, 3) for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:6]})
    top = sorted(range(len(data)), key=lambda i: -int(data[i][iW]))[:n]
    for i in sorted(top):
        r = data[i]
        rs = sorted(((int(r[h.index(c)] or 0), c[6:]) for c in reasons), reverse=True)[:2]
        print(f"{i:5d} {r[iW]:>5} {rs[0][1]}:{rs[0][0]} {rs[1][1]}:{rs[1][0]}  {r[iS][:80]}")
