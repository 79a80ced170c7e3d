"""Per-source-line warp instructions and stall samples of one kernel from
`ncu -i rep --page source --csv --print-source cuda,sass` (file argument):
SASS rows are summed into the source line above them; the line text is
taken from SRC (ncu's own attribution of the file path can be wrong when a
.cu file includes another).
python tools/ncu_src.py mix.csv SRC [N]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
src = open(sys.argv[2]).read().split("\n")
N = int(sys.argv[3]) if len(sys.argv) > 3 else 60


def num(v):
    try:
        return float(v.replace(",", ""))
    except ValueError:
        return 0.0


hdr = next(r for r in rows if r and r[0] == "Line No")
ist, iex = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
first = True
st = collections.Counter()
ins = collections.Counter()
line = None
for r in rows:
    if r and r[0] == "File Path":
        if not first:
            break  # the first file block only
        first = False
        continue
    if not r or r[0] in ("Line No", "Function Name"):
        continue
    if r[0].isdigit():
        line = int(r[0])
        continue
    if line is None or r[2] == "...":
        continue
    st[line] += num(r[ist])
    ins[line] += num(r[iex])
ts, te = sum(st.values()), sum(ins.values())
print("samples", ts, "warp-inst", te)
top = sorted(set(st) | set(ins), key=lambda l: -(st[l] / max(ts, 1) + ins[l] / max(te, 1)))[:N]
for l in sorted(top):
    print(f"{l:>5} {100*st[l]/max(ts,1):5.1f}%st {100*ins[l]/max(te,1):5.1f}%in  {src[l-1].strip()[:95] if l <= len(src) else ''}")
