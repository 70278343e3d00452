"""Per-task trace of the row-warp kernel (debug build, -DLCB_RW_DEBUG).

LCB_NVCC_EXTRA=-DLCB_RW_DEBUG python tools/debug_rw.py --conc 6 --rows 16
Prints S, ES, relmax, m, zmin, blo, bhi, nb, nl, ovf per task (first 256).
"""

from __future__ import annotations

import argparse
import ctypes as C
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
    ap.add_argument("--rows", type=int, default=16)
    ap.add_argument("--conc", type=float, default=2.5)
    ap.add_argument("--top-p", type=float, default=0.9)
    ap.add_argument("--fp32", action="store_true")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    dt = torch.float32 if a.fp32 else torch.bfloat16
    n = a.rows
    states = _dev.u64_tensor([mix2(7, i) for i in range(n)], dev)
    rows = torch.empty((n, a.V), dtype=dt, device=dev)
    _capi.check(_capi.lib.lc_fill_logits(states.data_ptr(), n, a.V, a.conc, 5.0,
                                         _capi.LC_F32 if a.fp32 else _capi.LC_BF16, rows.data_ptr(), a.V, None))
    tasks = lcb.make_tasks(row=np.arange(n), pos=np.zeros(n), temperature=0.6, top_k=0, top_p=a.top_p,
                           draw_begin=np.arange(n) * 4, draw_end=np.arange(n) * 4 + 4, seed_base=np.arange(n) * 4)
    tt = torch.from_numpy(tasks.view(np.uint8).copy()).to(dev)
    seeds = _dev.u64_tensor([mix2(1, b) for b in range(4 * n)], dev)
    cnt = torch.zeros(8, dtype=torch.int64, device=dev)
    lcb.resample(rows, tt, seeds=seeds, n_draws=4 * n, counters=cnt)
    torch.cuda.synchronize()
    out = np.zeros((256, 12))
    f = _capi.lib.lcb_debug_fetch
    f.argtypes = [C.c_void_p]
    assert f(out.ctypes.data) == 0
    print("counters", cnt.cpu().tolist())
    print("   S            ES          relmax     m        zmin    blo  bhi  nb   nl  ovf")
    for i in range(min(n, 256)):
        r = out[i]
        print(f"{r[0]:12.6g} {r[1]:11.4g} {r[2]:10.3g} {r[3]:8.4f} {r[4]:8.4f} {r[5]:4.0f} {r[6]:4.0f} "
              f"{r[7]:4.0f} {r[8]:5.0f} {r[9]:2.0f}")


if __name__ == "__main__":
    main()
