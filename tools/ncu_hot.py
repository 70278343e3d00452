"""Hot CUDA source lines of an ncu report: samples and instructions executed per line.

python tools/ncu_hot.py gpurun_out/x.ncu-rep [N]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True).stdout.decode("utf-8", "replace")
fn, hdr, agg = None, None, []
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fn = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = {k: i for i, k in enumerate(r)}
        continue
    if hdr and r[0] not in ("", "Function Name"):
        try:
            agg.append((int(r[hdr["# Samples"]]), int(r[hdr["Instructions Executed"]]), fn, r[0], r[1][:90]))
        except (ValueError, IndexError):
            pass
tot = sum(a[0] for a in agg) or 1
toti = sum(a[1] for a in agg) or 1
for s, i, f, ln, src in sorted(agg, reverse=True)[:n]:
    print(f"{100 * s / tot:5.1f}% smp {100 * i / toti:5.1f}% ins  {f}:{ln}  {src}")
