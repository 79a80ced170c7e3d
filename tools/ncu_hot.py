"""Top SASS instructions by warp-stall samples from an ncu --page source
--print-source sass CSV (stdin).  python tools/ncu_hot.py [N] < sass.csv"""
import csv
import sys

rows = list(csv.reader(sys.stdin))
hdr = rows[1]
data = [r for r in rows[2:] if len(r) == len(hdr) and r[0] != "Address"]
ia, isrc, ist = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
tot = sum(int(r[ist] or 0) for r in data if r[ist].isdigit())
data = [r for r in data if r[ist].isdigit()]
n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
print("total samples", tot)
order = sorted(range(len(data)), key=lambda i: -int(data[i][ist] or 0))[:n]
for i in sorted(order):
    r = data[i]
    print(f"{i:5d} {int(r[ist]):7d} {100*int(r[ist])/tot:5.1f}%  {r[isrc].strip()[:90]}")
