"""Summarise an ncu source-page CSV: stall reasons in total and the hottest SASS lines.

    ncu -i rep --page source --csv --print-source sass > x.csv; python tools/ncu_src.py x.csv [top]
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hdr = rows[1]
data = [r for r in rows[2:] if len(r) == len(hdr)]
i_src, i_s = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = {h: 0 for h in reasons}
for r in data:
    for h in reasons:
        v = r[hdr.index(h)]
        tot[h] += int(v) if v.isdigit() else 0
allsum = sum(tot.values())
print("samples", allsum)
for h, v in sorted(tot.items(), key=lambda x: -x[1])[:10]:
    print(f"  {h:28s} {v:8d} {100.0 * v / max(allsum, 1):5.1f}%")
print("hottest instructions:")
data.sort(key=lambda r: -int(r[i_s]) if r[i_s].isdigit() else 0)
for r in data[:top]:
    det = sorted(((int(r[hdr.index(h)]) if r[hdr.index(h)].isdigit() else 0, h[6:]) for h in reasons), reverse=True)[:2]
    print(f"  {r[i_s]:>6s}  {r[i_src].strip()[:60]:60s} {det}")
