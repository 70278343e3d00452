"""Copy one GPU round's outputs (tools/gpu_round.sh) from gpurun_out/ into profiles/ under a tag,
with ncu summaries (key metrics, stall reasons, hot source lines) and the C2 launch list.

python tools/collect_round.py r1_final
"""
import collections
import csv
import io
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
O = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")
tag = sys.argv[1] if len(sys.argv) > 1 else "round"

for name in ["bench_c2", "bench_ref", "bench_c1", "bench_c3", "bench_c5", "bench_c4", "bench_c1h", "bench_c2w"]:
    f = os.path.join(O, name + ".json")
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print("skip", name, e)
        continue
    json.dump(d, open(os.path.join(P, f"{tag}_{name}.json"), "w"), indent=1)
for name in ["c3_sweep.jsonl", "pytest_gpu.log", "smoke.log"]:
    if os.path.exists(os.path.join(O, name)):
        shutil.copy(os.path.join(O, name), os.path.join(P, f"{tag}_{name}"))

lf = os.path.join(O, "launches.csv")
if os.path.exists(lf):
    rows = [r for r in csv.reader(open(lf)) if len(r) > 10]
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.OrderedDict()
    for r in rows[1:]:
        agg.setdefault(r[ki].split("(")[0].replace("void ", ""), []).append(float(r[vi].replace(",", "")) / 1e3)
    tot = sum(sum(v) for v in agg.values())
    with open(os.path.join(P, f"{tag}_launches_c2.txt"), "w") as f:
        for k, v in agg.items():
            f.write(f"{k[:60]:60s} n={len(v):4d} total={sum(v):10.1f} us  avg={sum(v)/len(v):9.1f} us  "
                    f"share={100*sum(v)/tot:5.1f}%\n")

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
for rep in ["stage", "wide", "rowwarp"]:
    f = os.path.join(O, rep + ".ncu-rep")
    if not os.path.exists(f):
        continue
    out = subprocess.run(["ncu", "-i", f, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hh, units, vv = r[0], r[1], r[2] if len(r) > 2 else r[1]
    d = {k: f"{v} {u}" for k, u, v in zip(hh, units, vv) if k in WANT}
    st = []
    for k, x in zip(hh, vv):
        if "pcsamp_warps_issue_stalled" in k and "not_issued" not in k:
            try:
                st.append((float(x.replace(",", "")), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    d["top_stalls"] = [f"{k}={int(a)}" for a, k in sorted(st, reverse=True)[:8]]
    json.dump(d, open(os.path.join(P, f"{tag}_ncu_{rep}.json"), "w"), indent=1)
    hot = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_hot.py"), f, "30"], capture_output=True,
                         text=True).stdout
    open(os.path.join(P, f"{tag}_ncu_{rep}_hotlines.txt"), "w").write(hot)
print("collected into profiles/ with tag", tag)
