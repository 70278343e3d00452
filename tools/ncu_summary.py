"""Summarise an ncu report (one kernel regex) into JSON for profiles/.

python tools/ncu_summary.py gpurun_out/prof.ncu-rep rowwarp > profiles/xxx.json
Reports per launch: duration, DRAM bytes read/written, DRAM throughput, IPC,
occupancy, registers, and the top warp-stall reasons.
"""

from __future__ import annotations

import csv
import io
import json
import subprocess
import sys


def raw(rep: str):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def main():
    rep, pat = sys.argv[1], sys.argv[2]
    hdr, units, data = raw(rep)
    idx = {n: i for i, n in enumerate(hdr)}
    want = {
        "duration_ns": "gpu__time_duration.sum",
        "dram_read_bytes": "dram__bytes_read.sum",
        "dram_write_bytes": "dram__bytes_write.sum",
        "dram_pct_peak": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "ipc": "sm__inst_executed.avg.per_cycle_active",
        "occupancy_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
        "registers": "launch__registers_per_thread",
        "grid": "launch__grid_size",
        "block": "launch__block_size",
    }
    out = []
    for r in data:
        name = r[idx["Kernel Name"]]
        if pat not in name:
            continue
        d = {"kernel": name[:120]}
        for k, m in want.items():
            if m in idx:
                u = units[idx[m]]
                v = r[idx[m]].replace(",", "")
                try:
                    x = float(v)
                except ValueError:
                    continue
                if u in ("Kbyte", "KB"):
                    x *= 1e3
                elif u == "Mbyte":
                    x *= 1e6
                elif u == "Gbyte":
                    x *= 1e9
                elif u in ("usecond", "us"):
                    x *= 1e3
                elif u in ("msecond", "ms"):
                    x *= 1e6
                elif u in ("byte", "B"):
                    pass
                d[k] = x
        stalls = {}
        for n, i in idx.items():
            if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("not_issued"):
                try:
                    stalls[n.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(r[i].replace(",", ""))
                except ValueError:
                    pass
        tot = sum(stalls.values()) or 1.0
        d["top_stalls_pct"] = {k: round(100 * v / tot, 1) for k, v in sorted(stalls.items(), key=lambda x: -x[1])[:6]}
        if "duration_ns" in d and "dram_read_bytes" in d:
            d["dram_gbs"] = (d["dram_read_bytes"] + d.get("dram_write_bytes", 0.0)) / d["duration_ns"]
            d["traffic_bytes"] = d["dram_read_bytes"] + d.get("dram_write_bytes", 0.0)
        out.append(d)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
