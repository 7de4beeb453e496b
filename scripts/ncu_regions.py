"""Stall samples of one kernel in an ncu capture, by SASS region and top instructions.
    python scripts/ncu_regions.py <rep> [topN]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
k = next(i for i, r in enumerate(rows) if "Address" in r)
hdr, data = rows[k], rows[k + 1:]
ia, isrc = hdr.index("Address"), hdr.index("Source")
iall = hdr.index("Warp Stall Sampling (All Samples)")
cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
ci = {c: hdr.index(c) for c in cols}
tot = sum(float(r[iall] or 0) for r in data)
print(f"samples {tot:.0f}")
agg = {c: sum(float(r[ci[c]] or 0) for r in data) for c in cols}
print(" ".join(f"{c[6:]}={v / tot:.2f}" for c, v in sorted(agg.items(), key=lambda x: -x[1]) if v / tot > 0.01))
items = sorted(((float(r[iall] or 0), r) for r in data), key=lambda x: -x[0])
for v, r in items[:top]:
    t2 = sorted(((float(r[ci[c]] or 0), c) for c in cols), reverse=True)[:2]
    print(f"{v / tot:.3f} {r[ia][-5:]} {r[isrc].strip()[:64]:64s} {t2[0][1][6:]}:{t2[0][0]:.0f} {t2[1][1][6:]}:{t2[1][0]:.0f}")
