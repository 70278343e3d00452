"""Bulk parity check of whole benchmark steps against the oracle (TEST INFRASTRUCTURE ONLY).

Used by ``bench.py --check`` (the untimed validation leg) and by the tests: every
token a GPU step drew, and every task's kept-set size, is recomputed here from
the same rows and the same uniforms with the oracle restatement of
``sample(truncate(softmax(z, T), k, p), stream)`` (sampling.py:57-109), on all
host cores.  Rows are regenerated with the reference producer
(``fill_logits``, kernels.py:47-60; bf16-rounded for bf16 slabs, as the GPU
stores them); uniforms are ``RngStream(seed).next_float()`` at the draw number
(mixing.py:81-98).

Per row the oracle computes p, the kept order and q once
(``kept_order_fast`` / ``draw_many``: the same values the per-draw reference
path computes on every call), then checks all draws of that row.
"""

from __future__ import annotations

import numpy as np

from . import mixing_ref, sampling_ref


def check_rows(job) -> dict:
    """job: dict(V, T, k, p, bf16, conc, states [n] u64, seeds [n, D] u64 (the seed of each of
    the row's D draws), index [n] (the draw number of the row's draws), tokens [n, D] i32,
    kept [n] i32 or None).  Returns counts and up to 8 mismatch examples."""
    V, T, k, p = job["V"], job["T"], job["k"], job["p"]
    out = {"rows": 0, "draws": 0, "token_mismatches": 0, "kept_checked": 0, "kept_mismatches": 0,
           "examples": []}
    kept = job.get("kept")
    for i, st in enumerate(job["states"]):
        z = mixing_ref.fill_logits_np(int(st), V, job["conc"], 5.0)
        if job["bf16"]:
            z = mixing_ref.bf16_round(z)
        prob = sampling_ref.softmax(z, T)
        q, K = sampling_ref.truncate_fast(prob, k, p)
        us = mixing_ref.uniforms_np(job["seeds"][i], np.full(len(job["seeds"][i]), int(job["index"][i])))
        want = sampling_ref.draw_many(q, us)
        got = np.asarray(job["tokens"][i])
        bad = np.flatnonzero(got != want)
        out["rows"] += 1
        out["draws"] += len(want)
        out["token_mismatches"] += len(bad)
        if len(bad) and len(out["examples"]) < 8:
            out["examples"].append({"row": int(job.get("row_ids", range(len(job["states"])))[i]),
                                    "draw": int(bad[0]), "got": int(got[bad[0]]), "want": int(want[bad[0]])})
        if kept is not None:
            Kg = int(kept[i])
            ok = Kg == K
            if ok and K < V:  # identity rows (K == V) keep every id: nothing more to compare
                ids = _zorder_prefix(z, K)
                ok = np.array_equal(np.sort(ids[prob[ids] > 0]), np.flatnonzero(q > 0))
            out["kept_checked"] += 1
            if not ok:
                out["kept_mismatches"] += 1
                if len(out["examples"]) < 8:
                    out["examples"].append({"row": int(job.get("row_ids", range(len(job["states"])))[i]),
                                            "kept_got": Kg, "kept_want": int(K)})
    return out


def _zorder_prefix(z, K):
    """First K ids in (logit desc, id asc) order: the kernels' kept-set description."""
    z = np.asarray(z, dtype=np.float64)
    if K <= 0:
        return np.zeros(0, np.int64)
    if K >= len(z):
        return np.lexsort((np.arange(len(z)), -z))
    thr = z[np.argpartition(-z, K - 1)[:K]].min()
    cand = np.flatnonzero(z >= thr)
    return cand[np.lexsort((cand, -z[cand]))][:K]


def merge(results) -> dict:
    tot = {"rows": 0, "draws": 0, "token_mismatches": 0, "kept_checked": 0, "kept_mismatches": 0, "examples": []}
    for r in results:
        for key in ("rows", "draws", "token_mismatches", "kept_checked", "kept_mismatches"):
            tot[key] += r[key]
        tot["examples"] += r["examples"][: max(0, 8 - len(tot["examples"]))]
    return tot
