"""Aggregate an ncu source page (--print-source=cuda,sass CSV) by CUDA source line."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
fn = None
func = None
agg = {}
hdr = None
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
    if hdr is None or len(r) < len(hdr):
        continue
    if r[0].isdigit():
        key = (func, fn, int(r[0]), r[1][:90])
        try:
            s, n = int(r[wi] or 0), int(r[ii] or 0)
        except ValueError:
            continue
        a = agg.setdefault(key, [0, 0])
        a[0] += s
        a[1] += n
flt = sys.argv[2] if len(sys.argv) > 2 else ""
items = [(k, v) for k, v in agg.items() if flt in k[0]]
tot = sum(v[0] for _, v in items) or 1
toti = sum(v[1] for _, v in items) or 1
print(f"samples {tot} instructions {toti}")
for k, v in sorted(items, key=lambda x: -x[1][0])[: int(sys.argv[3]) if len(sys.argv) > 3 else 40]:
    print(f"{v[0]:7d} {100 * v[0] / tot:5.1f}%  {v[1]:11d} {100 * v[1] / toti:5.1f}%  {k[1]}:{k[2]}  {k[3]}")
