"""Per-instruction stall samples of the step loop from an ncu source-page CSV
(ncu -i <rep> --page source --csv --print-source sass > x.csv).
    python scripts/srcstall.py x.csv"""
import csv, re, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]; data = rows[2:]
ia, isrc = hdr.index("Address"), hdr.index("Source")
iall = hdr.index("Warp Stall Sampling (All Samples)")
cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
ci = {c: hdr.index(c) for c in cols}
tot = sum(float(r[iall] or 0) for r in data)
# innermost loop containing a VOTE: the backward branch closing it
best = None
for k, r in enumerate(data):
    m = re.search(r"BRA.*?(0x[0-9a-f]+)", r[isrc])
    if not m:
        continue
    tgt = int(m.group(1), 16)
    if tgt >= int(r[ia], 16):
        continue
    s = next((j for j, x in enumerate(data) if int(x[ia], 16) == tgt), None)
    if s is None:
        continue
    body = data[s:k + 1]
    if any("VOTE" in x[isrc] for x in body) and sum("LDS" in x[isrc] for x in body) >= 16 and \
            not any("LDG" in x[isrc] for x in body):
        if best is None or len(body) < len(best):
            best = body
lt = sum(float(r[iall] or 0) for r in best)
print(f"samples total {tot:.0f}, loop {lt:.0f} ({lt / tot:.2f}), loop instrs {len(best)}")
agg = {c: sum(float(r[ci[c]] or 0) for r in best) for c in cols}
print(" ".join(f"{c[6:]}={v / lt:.2f}" for c, v in sorted(agg.items(), key=lambda x: -x[1]) if v / lt > 0.01))
for r in best:
    v = float(r[iall] or 0)
    top = sorted(((float(r[ci[c]] or 0), c) for c in cols), reverse=True)[:2]
    print(f"{v:6.0f} {r[isrc].strip()[:58]:58s} {top[0][1][6:]}:{top[0][0]:.0f} {top[1][1][6:]}:{top[1][0]:.0f}")
