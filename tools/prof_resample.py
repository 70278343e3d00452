"""Standalone driver for profiling the resample kernel (ncu target).

python tools/prof_resample.py --V 32000 --rows 4096 --draws 32 --top-p 0.9 --bf16 --iters 3
Prints per-call CUDA-event times and the tier/reason counters
(0 requeued tasks, 1 unresolved draws, 2 bad rows, 3 small-cut uncertain,
4 large-nucleus uncertain, 5 draw uncertain, 7 candidate/scratch overflow).
"""

from __future__ import annotations

import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_17353_b200 as lcb  # noqa: E402
from paper_2604_17353_b200 import _capi, _dev  # noqa: E402
from paper_2604_17353_b200.mixing import mix2  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--V", type=int, default=32000)
    ap.add_argument("--rows", type=int, default=4096)
    ap.add_argument("--draws", type=int, default=32)
    ap.add_argument("--T", type=float, default=0.6)
    ap.add_argument("--top-k", type=int, default=0)
    ap.add_argument("--top-p", type=float, default=0.9)
    ap.add_argument("--conc", type=float, default=2.5)
    ap.add_argument("--bf16", action="store_true")
    ap.add_argument("--iters", type=int, default=3)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    dt = torch.bfloat16 if a.bf16 else torch.float32
    states = _dev.u64_tensor([mix2(7, i) for i in range(a.rows)], dev)
    rows = torch.empty((a.rows, a.V), dtype=dt, device=dev)
    _capi.check(_capi.lib.lc_fill_logits(states.data_ptr(), a.rows, a.V, a.conc, 5.0,
                                         _capi.LC_BF16 if a.bf16 else _capi.LC_F32, rows.data_ptr(), a.V, None))
    n = a.rows
    tasks = lcb.make_tasks(row=np.arange(n), pos=np.arange(n) % 500, temperature=a.T, top_k=a.top_k, top_p=a.top_p,
                           draw_begin=np.arange(n) * a.draws, draw_end=np.arange(n) * a.draws + a.draws,
                           seed_base=np.arange(n) % 256 * a.draws)
    tt = torch.from_numpy(tasks.view(np.uint8).copy()).to(dev)
    seeds = _dev.u64_tensor([mix2(1, b) for b in range(256 * a.draws)], dev)
    cnt = torch.zeros(8, dtype=torch.int64, device=dev)
    for i in range(a.iters):
        cnt.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        tok_out = torch.full((n * a.draws,), -7, dtype=torch.int32, device=dev)
        fl_out = torch.zeros(n * a.draws, dtype=torch.uint8, device=dev)
        lcb.resample(rows, tt, seeds=seeds, n_draws=n * a.draws, counters=cnt, out=(tok_out, fl_out))
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e)
        gb = n * a.V * rows.element_size() / 1e9
        print(f"iter {i}: {ms:.3f} ms  {n / ms / 1e3:.2f} M rows/s  {gb / ms * 1e3:.1f} GB/s  "
              f"counters {cnt.cpu().tolist()}  unwritten {int((tok_out == -7).sum())}", flush=True)
        if os.environ.get("LCB_STAGE_PROF") == "1":
            import ctypes
            buf = (ctypes.c_ulonglong * 12)()
            if _capi.lib.lcb_stage_prof_fetch(buf) == 0:
                ph = list(buf)
                if a.V > 32000:  # wide top-k kernel: 0 wait, 1 max, 2 threshold, 3 mass, 4 list, 5 final, 6 rows
                    r_ = max(ph[6], 1)
                    print("  wide phases, clks per row: " + "  ".join(
                        f"{nm}={ph[k] / r_:.0f}" for k, nm in enumerate(["wait", "max", "thr", "mass", "list",
                                                                      "final"])) + f"  rows={ph[6]}", flush=True)
                    continue
                rows_, big = max(ph[9], 1), max(ph[10], 1)
                names = ["wait", "A", "B", "fastfin", "H", "cls+cut", "C", "D", "end"]
                print("  stage phases, clks per row (per big row for H..D): " + "  ".join(
                    f"{nm}={ph[k] / (big if 4 <= k <= 7 else rows_):.0f}" for k, nm in enumerate(names))
                    + f"  pop={ph[11] / rows_:.0f}  rows={ph[9]} big={ph[10]}", flush=True)


if __name__ == "__main__":
    main()
