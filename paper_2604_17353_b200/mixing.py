"""64-bit mixing primitives (reference pkg/src/agentserve/mixing.py:43-105).

Scalar helpers (``avalanche64``, ``mix2``, ``RngStream``) are the definitions
callers use to derive seeds (e.g. the flow runtime's ``mix2(run_seed, n)``,
flow.py:474); the hot-path work -- hashing thousands of prompts and drawing
uniforms for every replayed position -- runs on the GPU through
``hash_prompts`` / ``uniforms`` (liblcb200 ``lc_hash_prefix`` / ``lc_uniforms``).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _capi, _dev

MASK64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15
EMPTY_HASH = 0xA0761D6478BD642F
PEAK_SALT = 0x8BB84B93962EACC9
SAMPLER_SALT = 0x2545F4914F6CDD1D
SCORE_SALT = 0x6A09E667F3BCC909


def avalanche64(z: int) -> int:
    z &= MASK64
    z ^= z >> 30
    z = (z * 0xBF58476D1CE4E5B9) & MASK64
    z ^= z >> 27
    z = (z * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def stream_u64(state: int, index: int) -> int:
    return avalanche64((state + (index + 1) * GOLDEN) & MASK64)


def unit_float(u: int) -> float:
    return (u >> 11) * 2.0 ** -53


def fold_token(h: int, token: int) -> int:
    return avalanche64(h ^ ((token + 1) & MASK64))


def mix2(a: int, b: int) -> int:
    return avalanche64(avalanche64(a) ^ (b & MASK64))


class RngStream:
    """Counter-based request stream (mixing.py:81-105): u_i depends only on (seed, i)."""

    __slots__ = ("_state", "position", "seed")

    def __init__(self, seed: int):
        self.seed = seed & MASK64
        self._state = avalanche64((seed ^ SAMPLER_SALT) & MASK64)
        self.position = 0

    def next_float(self) -> float:
        u = stream_u64(self._state, self.position)
        self.position += 1
        return unit_float(u)

    def fork(self, label: int) -> "RngStream":
        child = RngStream.__new__(RngStream)
        child.seed = None
        child._state = mix2(self._state, label)
        child.position = 0
        return child


def hash_prompts(prompts, parents=None, dev=None) -> torch.Tensor:
    """Digests of many prompts on the GPU (K2).  Returns an int64 tensor holding
    the uint64 bit patterns; ``parents`` extends existing digests (prefix
    extension, mixing.py:63-65)."""
    d = _dev.device(dev)
    lens = [len(p) for p in prompts]
    offs = np.zeros(len(prompts) + 1, dtype=np.int64)
    np.cumsum(lens, out=offs[1:])
    flat = np.concatenate([np.asarray(p, dtype=np.int32) for p in prompts]) if offs[-1] else np.zeros(1, np.int32)
    toks = torch.from_numpy(flat).to(d)
    offt = torch.from_numpy(offs).to(d)
    par = _dev.u64_tensor(parents, d) if parents is not None else None
    out = torch.empty(len(prompts), dtype=torch.int64, device=d)
    _capi.check(_capi.lib.lc_hash_prefix(toks.data_ptr(), offt.data_ptr(), _dev.ptr(par), len(prompts),
                                         out.data_ptr(), _dev.stream_ptr(d)), "lc_hash_prefix")
    return out


def hash_tokens(tokens, start: int = EMPTY_HASH) -> int:
    """Rolling hash of one token sequence, computed by the GPU hasher."""
    out = hash_prompts([list(tokens)], parents=[start])
    return int(_dev.u64_numpy(out)[0])


def uniforms(seeds, index, dev=None) -> torch.Tensor:
    """u[i] = RngStream(seeds[i]) draw number index[i], on the GPU (fp64)."""
    d = _dev.device(dev)
    s = _dev.u64_tensor(seeds, d)
    ix = _dev.to_dev(index, torch.int64, d)
    out = torch.empty(s.numel(), dtype=torch.float64, device=d)
    _capi.check(_capi.lib.lc_uniforms(s.data_ptr(), ix.data_ptr(), s.numel(), out.data_ptr(), _dev.stream_ptr(d)),
                "lc_uniforms")
    return out
