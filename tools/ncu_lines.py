"""Per-source-line instructions executed and warp-stall samples of one kernel
from `ncu -i rep --page source --csv --print-source cuda,sass` (stdin).
python tools/ncu_lines.py <function-substring> [N] < mix.csv"""
import csv
import sys

key = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
rows = list(csv.reader(sys.stdin))
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Function Name":
        cur = [r[1], []]
        blocks.append(cur)
    elif cur is not None:
        cur[1].append(r)
for name, rs in blocks:
    if key not in name:
        continue
    hdr = next(r for r in rs if r and r[0] == "Line No")
    ist, iex = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
    lines = [r for r in rs if r and r[0] not in ("", "Line No") and len(r) == len(hdr)]
    num = lambda v: int(v) if v.isdigit() else 0
    ts = sum(num(r[ist]) for r in lines)
    te = sum(num(r[iex]) for r in lines)
    print(name[:90], "samples", ts, "warp-inst", te)
    top = sorted(lines, key=lambda r: -num(r[ist]))[:N]
    for r in sorted(top, key=lambda r: int(r[0])):
        print(f"{r[0]:>5} {100*num(r[ist])/max(ts,1):5.1f}%st {100*num(r[iex])/max(te,1):5.1f}%in  {r[1].strip()[:100]}")
