"""Oracle restatement of the 64-bit mixing primitives (TEST INFRASTRUCTURE ONLY).

Restates ``agentserve/mixing.py`` (reference ``pkg/src/agentserve/mixing.py``)
and the normative contract ``pkg/docs/determinism.md:14-92``:

* ``avalanche64``      -- splitmix64 finalizer, mixing.py:43-50
* ``stream_u64``       -- mixing.py:53-55
* ``unit_float``       -- mixing.py:58-60
* ``fold_token`` / ``hash_tokens`` -- mixing.py:63-73
* ``mix2``             -- mixing.py:76-78
* request uniforms     -- ``RngStream`` mixing.py:81-98, determinism.md:78-92
* synthetic logits     -- kernels.py:47-60 / _mixcore.pyx:27-40,
  determinism.md:55-76 (the *producer* of benchmark rows, not the path)

Scalar functions use Python ints; the ``*_np`` variants are vectorised with
wrapping ``uint64`` numpy arithmetic and are checked bit-for-bit against the
scalar ones and against the reference's golden values in ``tests/``.
"""

from __future__ import annotations

import numpy as np

MASK64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15
MULT1 = 0xBF58476D1CE4E5B9
MULT2 = 0x94D049BB133111EB
EMPTY_HASH = 0xA0761D6478BD642F
PEAK_SALT = 0x8BB84B93962EACC9
SAMPLER_SALT = 0x2545F4914F6CDD1D

_U = np.uint64


def avalanche64(z: int) -> int:
    z &= MASK64
    z ^= z >> 30
    z = (z * MULT1) & MASK64
    z ^= z >> 27
    z = (z * MULT2) & MASK64
    return z ^ (z >> 31)


def stream_u64(state: int, index: int) -> int:
    return avalanche64((state + (index + 1) * GOLDEN) & MASK64)


def unit_float(u: int) -> float:
    return (u >> 11) * 2.0 ** -53


def fold_token(h: int, token: int) -> int:
    return avalanche64(h ^ ((token + 1) & MASK64))


def hash_tokens(tokens, start: int = EMPTY_HASH) -> int:
    h = start
    for t in tokens:
        h = fold_token(h, int(t))
    return h


def mix2(a: int, b: int) -> int:
    return avalanche64(avalanche64(a) ^ (b & MASK64))


def sampler_state(seed: int) -> int:
    """Root of a request's draw stream (mixing.py:92)."""
    return avalanche64((seed ^ SAMPLER_SALT) & MASK64)


def uniform(seed: int, index: int) -> float:
    """``RngStream(seed)``'s ``index``-th ``next_float()`` (mixing.py:95-98)."""
    return unit_float(stream_u64(sampler_state(seed), index))


# -- vectorised (wrapping uint64) ---------------------------------------------------


def avalanche64_np(z: np.ndarray) -> np.ndarray:
    z = np.asarray(z, dtype=np.uint64).copy()
    with np.errstate(over="ignore"):
        z ^= z >> _U(30)
        z *= _U(MULT1)
        z ^= z >> _U(27)
        z *= _U(MULT2)
        z ^= z >> _U(31)
    return z


def uniforms_np(seeds, positions) -> np.ndarray:
    """u[i] = uniform(seeds[i], positions[i]) for arrays of seeds/positions."""
    seeds = np.asarray(seeds, dtype=np.uint64)
    positions = np.asarray(positions, dtype=np.uint64)
    with np.errstate(over="ignore"):
        st = avalanche64_np(seeds ^ _U(SAMPLER_SALT))
        u = avalanche64_np(st + (positions + _U(1)) * _U(GOLDEN))
    return (u >> _U(11)).astype(np.float64) * 2.0 ** -53


def fill_logits_np(state: int, vocab: int, concentration: float, logit_range: float) -> np.ndarray:
    """Synthetic logits row (determinism.md:55-76; kernels.py:47-60)."""
    with np.errstate(over="ignore"):
        z = _U(state & MASK64) + np.arange(1, vocab + 1, dtype=np.uint64) * _U(GOLDEN)
    z = avalanche64_np(z)
    x = (z >> _U(11)).astype(np.float64) * 2.0 ** -53
    out = ((2.0 * x - 1.0) * logit_range).astype(np.float32)
    peak = avalanche64(state ^ PEAK_SALT) % vocab
    out[peak] = np.float32(out[peak] + np.float32(concentration * logit_range))
    return out


def fill_rows_np(states, vocab: int, concentration: float = 2.5, logit_range: float = 5.0) -> np.ndarray:
    return np.stack([fill_logits_np(int(s), vocab, concentration, logit_range) for s in states])


def bf16_round(x: np.ndarray) -> np.ndarray:
    """fp32 -> bf16 (round-to-nearest-even) -> fp32, as the GPU slab stores it."""
    b = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    rounding = ((b >> np.uint64(16)) & np.uint64(1)) + np.uint64(0x7FFF)
    nan = np.isnan(x)
    r = ((b + rounding) >> np.uint64(16)) << np.uint64(16)
    r = r.astype(np.uint32).view(np.float32)
    return np.where(nan, np.float32(np.nan), r).astype(np.float32)
