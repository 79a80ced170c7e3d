"""Stall-reason totals and top SASS lines with their dominant reasons from an
ncu --page source --csv --print-source sass export (stdin)."""
import csv
import sys

rows = list(csv.reader(sys.stdin))
hdr = rows[1]
data = [r for r in rows[2:] if len(r) == len(hdr) and r[0] != "Address"]
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
ri = [hdr.index(h) for h in reasons]
isrc = hdr.index("Source")
ist = hdr.index("Warp Stall Sampling (All Samples)")
num = lambda x: int(x) if x.isdigit() else 0
tot = {h: sum(num(r[i]) for r in data) for h, i in zip(reasons, ri)}
T = sum(tot.values()) or 1
print("stall totals:", ", ".join(f"{h[6:]}={100*v/T:.1f}%" for h, v in sorted(tot.items(), key=lambda kv: -kv[1]) if v))
n = int(sys.argv[1]) if len(sys.argv) > 1 else 20
order = sorted(range(len(data)), key=lambda i: -num(data[i][ist]))[:n]
for i in sorted(order):
    r = data[i]
    top = sorted(((num(r[j]), h[6:]) for h, j in zip(reasons, ri)), reverse=True)[:2]
    print(f"{i:5d} {num(r[ist]):6d}  {r[isrc].strip()[:60]:60s} {top}")
