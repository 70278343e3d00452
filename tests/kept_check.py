"""Kept-set check shared by the GPU tests and ``bench.py --check`` (TEST INFRASTRUCTURE).

The fused kernels report, per task, the size K of truncate()'s kept set
(``lc_draws.d_kept``); the set itself is then the first K ids of the row in
(logit desc, id asc) order -- the reference's ``lexsort((ids, -p))`` prefix
(sampling.py:80-94), because p is monotone in the logit.  The check rebuilds
that prefix from the row and compares it with the oracle:

* K equals ``len(kept_order)`` (V for the identity, sampling.py:78-79);
* the prefix's nonzero-probability ids equal ``flatnonzero(truncate(p) > 0)``
  (the golden ``kept`` arrays are exactly that).
"""

from __future__ import annotations

import numpy as np

from oracle import sampling_ref


def zorder_prefix(z: np.ndarray, K: int) -> np.ndarray:
    """The first K ids of z in (logit desc, id asc) order."""
    z = np.asarray(z, dtype=np.float64)
    if K >= len(z):
        return np.lexsort((np.arange(len(z)), -z))
    # (K small: partition first, then order the candidates exactly, ties by id)
    part = np.argpartition(-z, K - 1)[:K] if K > 0 else np.zeros(0, np.int64)
    if K == 0:
        return part
    thr = z[part].min()
    cand = np.flatnonzero(z >= thr)
    return cand[np.lexsort((cand, -z[cand]))][:K]


def kept_mismatch(z, T, top_k, top_p, K, p=None) -> str | None:
    """None when the kernel's kept count K describes the reference's kept set, else why not."""
    p = sampling_ref.softmax(z, T) if p is None else p
    order = sampling_ref.kept_order(p, top_k, top_p)
    want_len = len(z) if order is None else len(order)
    if int(K) != want_len:
        return f"K={int(K)} vs len(kept_order)={want_len}"
    got = zorder_prefix(z, int(K))
    got_nz = np.sort(got[p[got] > 0])
    want_nz = np.flatnonzero(p > 0) if order is None else np.sort(order[p[order] > 0])
    if not np.array_equal(got_nz, want_nz):
        return f"kept ids differ ({len(got_nz)} vs {len(want_nz)})"
    return None
