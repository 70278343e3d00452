"""Oracle restatement of the reference sampler (TEST INFRASTRUCTURE ONLY).

Restates ``pkg/src/agentserve/sampling.py`` with the *same numpy operation
order*, because token decisions must be bit-identical to the reference given
the same uniforms:

* temperature softmax   -- sampling.py:57-68  (f64 divide, subtract max,
  ``np.exp``, divide by numpy's pairwise ``sum``; T == 0 -> one-hot at the
  first argmax)
* top-k / top-p         -- sampling.py:71-94  (lexsort by (-p, id); top-k only
  when ``k < V``; nucleus mass measured on the *untruncated* distribution with
  a sequential ``cumsum`` and ``searchsorted(..., 'left')``; renormalise by the
  pairwise sum of the kept probabilities taken in sorted order)
* inverse-CDF draw      -- sampling.py:97-109 (pairwise ``sum``, sequential
  ``cumsum`` in token-id order, ``searchsorted(u*total, 'right')``, clamp to
  V-1, back off over zero-probability tokens; zero mass -> RuntimeError)
* hotspot scores        -- sampling.py:112-160

The uniform ``u`` is passed explicitly instead of through ``RngStream``
(``sample`` only ever calls ``stream.next_float()`` once, sampling.py:99).
"""

from __future__ import annotations

import numpy as np


def softmax(z: np.ndarray, temperature: float) -> np.ndarray:
    n = len(z)
    if temperature == 0.0:
        out = np.zeros(n, dtype=np.float64)
        out[int(np.argmax(z))] = 1.0
        return out
    s = z.astype(np.float64) / temperature
    s -= s.max()
    e = np.exp(s)
    return e / e.sum()


def sorted_order(p: np.ndarray) -> np.ndarray:
    """Descending probability, ascending token id among equal probabilities."""
    return np.lexsort((np.arange(len(p)), -p))


def kept_order(p: np.ndarray, top_k, top_p: float) -> np.ndarray | None:
    """Token ids that survive truncation, in sorted order; None = identity."""
    if top_k is None and top_p == 1.0:
        return None
    order = sorted_order(p)
    if top_k is not None and top_k < len(p):
        order = order[:top_k]
    if top_p < 1.0:
        mass = np.cumsum(p[order])
        order = order[: int(np.searchsorted(mass, top_p, side="left")) + 1]
    return order


def kept_order_fast(p: np.ndarray, top_k, top_p: float, cand: int = 8192) -> np.ndarray | None:
    """``kept_order`` without the full O(V log V) lexsort (for bulk checks; equal by
    construction and pinned against ``kept_order`` in tests/test_oracle.py).

    The kept set is a prefix of the (p desc, id asc) order.  Every id outside
    C = {p >= theta} (theta = the m-th largest p) sorts after every id of C, so when
    the prefix ends inside C's sorted order -- top-k with k <= |C|, or the csum over
    C reaching top_p -- it is C's prefix: same ids, same order, and the sequential
    csum over it is the same sequence of additions.  Otherwise fall back to the full sort."""
    V = len(p)
    if top_k is None and top_p == 1.0:
        return None
    k = top_k if (top_k is not None and top_k < V) else None
    m = min(V, max(cand, k or 0))
    if m < V:
        theta = np.partition(p, V - m)[V - m]
        ids = np.flatnonzero(p >= theta)
        ids = ids[np.argsort(-p[ids], kind="stable")]  # (p desc, id asc): ids ascend into the sort
        if k is not None:
            ids = ids[:k]
        if top_p < 1.0:
            mass = np.cumsum(p[ids])
            j = int(np.searchsorted(mass, top_p, side="left"))
            if j < len(ids):
                return ids[: j + 1]
            if k is not None and len(ids) == k:
                return ids  # the top-k survivors never reach top_p: all kept
        elif k is not None:
            return ids
    return kept_order(p, top_k, top_p)


def draw_many(q: np.ndarray, us) -> np.ndarray:
    """``[draw(q, u) for u in us]`` with the total and cdf computed once (the same values
    ``draw`` computes on every call: numpy's pairwise sum and sequential cumsum)."""
    total = float(q.sum())
    if total <= 0.0:
        raise RuntimeError("sample() called with no probability mass")
    cdf = np.cumsum(q)
    idx = np.searchsorted(cdf, np.asarray(us, dtype=np.float64) * total, side="right")
    idx = np.minimum(idx, len(q) - 1)
    out = idx.copy()
    nz = np.flatnonzero(q != 0.0)
    # back off over zero-probability ids: the last nonzero id <= idx (id 0 if none)
    pos = np.searchsorted(nz, idx, side="right") - 1
    back = q[idx] == 0.0
    out[back] = np.where(pos[back] >= 0, nz[np.maximum(pos[back], 0)], 0)
    return out


def truncate_fast(p: np.ndarray, top_k=None, top_p: float = 1.0) -> tuple[np.ndarray, int]:
    """(truncate(p, top_k, top_p), len(kept_order) or V) via ``kept_order_fast``."""
    order = kept_order_fast(p, top_k, top_p)
    if order is None:
        return p, len(p)
    q = np.zeros(len(p), dtype=np.float64)
    kept = p[order]
    q[order] = kept / kept.sum()
    return q, len(order)


def truncate(p: np.ndarray, top_k=None, top_p: float = 1.0) -> np.ndarray:
    order = kept_order(p, top_k, top_p)
    if order is None:
        return p
    q = np.zeros(len(p), dtype=np.float64)
    kept = p[order]
    q[order] = kept / kept.sum()
    return q


def draw(q: np.ndarray, u: float) -> int:
    total = float(q.sum())
    if total <= 0.0:
        raise RuntimeError("sample() called with no probability mass")
    cdf = np.cumsum(q)
    i = int(np.searchsorted(cdf, u * total, side="right"))
    if i >= len(q):
        i = len(q) - 1
    while i > 0 and q[i] == 0.0:
        i -= 1
    return i


def resample(z: np.ndarray, temperature: float, top_k, top_p: float, u: float) -> int:
    """``sample(truncate(softmax(z, T), k, p), stream)`` with the draw ``u``."""
    return draw(truncate(softmax(z, temperature), top_k, top_p), u)


def resample_full(z, temperature, top_k, top_p, u):
    """Token, kept id set (nonzero truncated probabilities, ascending) and q."""
    q = truncate(softmax(z, temperature), top_k, top_p)
    return draw(q, u), np.flatnonzero(q > 0.0), q


# -- hotspot scoring (sampling.py:112-160) ------------------------------------------


def entropy(p: np.ndarray) -> float:
    nz = p[p > 0]
    return float(-(nz * np.log(nz)).sum())


def hotspot_score(p: np.ndarray, step: int, decay: float) -> float:
    return entropy(p) * (1.0 - float(p.max())) / (1.0 + decay * step)


def select_hotspots(scores: np.ndarray, threshold: float, max_hotspots=None) -> tuple:
    span = scores.max() - scores.min()
    if span == 0.0:
        return ()
    norm = (scores - scores.min()) / span
    pos = np.nonzero(norm > threshold)[0]
    if max_hotspots is not None and len(pos) > max_hotspots:
        pos = sorted(pos, key=lambda t: (-norm[t], t))[:max_hotspots]
    return tuple(sorted(int(t) for t in pos))


def row_scores(rows, temperature: float, decay: float) -> np.ndarray:
    return np.array([hotspot_score(softmax(z, temperature), t, decay) for t, z in enumerate(rows)])


def identify_hotspots(rows, temperature, decay, threshold, max_hotspots=None) -> tuple:
    if len(rows) == 0:
        raise ValueError("logits_seq must be non-empty")
    return select_hotspots(row_scores(rows, temperature, decay), threshold, max_hotspots)
