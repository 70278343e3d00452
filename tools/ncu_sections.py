"""Aggregate an ncu source page by '// ----' sections of lc_resample.cu."""
import csv
import re
import sys

src = open(sys.argv[2]).read().splitlines()
marks = []
for i, line in enumerate(src, 1):
    m = re.match(r"\s*// -{4,}\s*(.*)", line) or re.match(r"\s*// =+\s*(.*?)\s*=*$", line)
    if m:
        marks.append((i, m.group(1)[:50]))
    if re.match(r"(template|__device__|__global__)", line):
        marks.append((i, "fn:" + line[:50]))


def section(ln):
    name = "head"
    for i, n in marks:
        if i <= ln:
            name = n
        else:
            break
    return name


rows = list(csv.reader(open(sys.argv[1])))
agg = {}
hdr = None
fn = func = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fn = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        func = r[1]
        continue
    if r[0] == "Line No":
        hdr = r
        wi = hdr.index("Warp Stall Sampling (All Samples)")
        ii = hdr.index("Instructions Executed")
        continue
    if hdr is None or len(r) < len(hdr) or not r[0].isdigit() or "rowwarp" not in (func or ""):
        continue
    key = section(int(r[0])) if fn == "lc_resample.cu" else "lib:" + fn
    a = agg.setdefault(key, [0, 0])
    try:
        a[0] += int(r[wi] or 0)
        a[1] += int(r[ii] or 0)
    except ValueError:
        pass
ts = sum(v[0] for v in agg.values()) or 1
ti = sum(v[1] for v in agg.values()) or 1
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{100 * v[1] / ti:5.1f}% instr  {100 * v[0] / ts:5.1f}% stalls  {k}")
