"""Sampling interface of the reference (pkg/src/agentserve/sampling.py), on the GPU.

Drop-in functions keep the reference's names, argument meaning and error
behaviour (numpy arrays in, numpy arrays / ints out):

* ``softmax``        sampling.py:57-68   -> ``lc_softmax``
* ``truncate``       sampling.py:71-94   -> ``lc_truncate_probs``
* ``sample``         sampling.py:97-109  -> ``lc_draw_probs`` (one ``stream.next_float()``)
* ``entropy`` / ``max_prob`` / ``hotspot_score`` / ``select_hotspots`` /
  ``identify_hotspots``  sampling.py:112-160 (per-row scores by ``lc_row_entropy``)

The hot path is the fused ``resample`` (``lc_resample``): temperature ->
softmax -> top-k/top-p -> inverse-CDF draw for a batch of device-resident rows,
never materialising probabilities.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _capi, _dev
from .errors import ConfigError


@dataclass(frozen=True)
class SamplingConfig:
    temperature: float = 1.0
    top_k: int | None = None
    top_p: float = 1.0
    max_tokens: int = 16
    seed: int = 0

    def __post_init__(self):  # sampling.py:26-35
        if self.temperature < 0:
            raise ConfigError(f"temperature must be >= 0, got {self.temperature}")
        if not (0 < self.top_p <= 1):
            raise ConfigError(f"top_p must be in (0, 1], got {self.top_p}")
        if self.max_tokens < 1:
            raise ConfigError(f"max_tokens must be >= 1, got {self.max_tokens}")
        if self.top_k is not None and self.top_k < 1:
            raise ConfigError(f"top_k must be >= 1 when set, got {self.top_k}")


@dataclass(frozen=True)
class HotspotParams:
    decay: float = 0.01
    threshold: float = 0.6
    max_hotspots: int | None = None

    def __post_init__(self):  # sampling.py:47-51
        if self.decay < 0:
            raise ConfigError(f"decay must be >= 0, got {self.decay}")
        if not (0 <= self.threshold <= 1):
            raise ConfigError(f"threshold must be in [0, 1], got {self.threshold}")

    def cache_key(self, temperature: float) -> tuple:
        return (temperature, self.decay, self.threshold, self.max_hotspots)


def _rows_to_dev(rows, dev):
    """(n, V) float32/bf16 rows on the device plus the ABI dtype code."""
    if isinstance(rows, torch.Tensor):
        t = rows.to(dev)
        if t.dtype == torch.bfloat16:
            return t.contiguous(), _capi.LC_BF16
        return t.to(torch.float32).contiguous(), _capi.LC_F32
    a = np.asarray(rows, dtype=np.float32)
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev), _capi.LC_F32


def softmax(logits, temperature: float) -> np.ndarray:
    d = _dev.device()
    z, dt = _rows_to_dev(np.asarray(logits).reshape(1, -1) if not isinstance(logits, torch.Tensor)
                         else logits.reshape(1, -1), d)
    V = z.shape[1]
    out = torch.empty((1, V), dtype=torch.float64, device=d)
    temp = torch.tensor([float(temperature)], dtype=torch.float64, device=d)
    _capi.check(_capi.lib.lc_softmax(z.data_ptr(), dt, V, V, 1, temp.data_ptr(), out.data_ptr(), _dev.stream_ptr(d)),
                "lc_softmax")
    return out[0].cpu().numpy()


def truncate(probs: np.ndarray, top_k: int | None = None, top_p: float = 1.0) -> np.ndarray:
    if top_k is None and top_p == 1.0:
        return probs  # sampling.py:78-79 returns its input untouched
    d = _dev.device()
    p = torch.as_tensor(np.asarray(probs, dtype=np.float64)).reshape(1, -1).to(d)
    V = p.shape[1]
    out = torch.empty_like(p)
    scratch = torch.empty(V * 12 + 512, dtype=torch.uint8, device=d)
    _capi.check(_capi.lib.lc_truncate_probs(p.data_ptr(), V, 1, V, -1 if top_k is None else int(top_k),
                                            float(top_p), out.data_ptr(), scratch.data_ptr(), _dev.stream_ptr(d)),
                "lc_truncate_probs")
    return out[0].cpu().numpy()


def sample(probs: np.ndarray, stream) -> int:
    """Inverse-CDF draw; consumes exactly one stream value (sampling.py:97-109)."""
    u = stream.next_float()
    d = _dev.device()
    p = torch.as_tensor(np.asarray(probs, dtype=np.float64)).reshape(1, -1).to(d)
    ut = torch.tensor([u], dtype=torch.float64, device=d)
    tok = torch.empty(1, dtype=torch.int32, device=d)
    fl = torch.empty(1, dtype=torch.uint8, device=d)
    V = p.shape[1]
    _capi.check(_capi.lib.lc_draw_probs(p.data_ptr(), V, 1, V, ut.data_ptr(), tok.data_ptr(), fl.data_ptr(),
                                        _dev.stream_ptr(d)), "lc_draw_probs")
    if int(fl.item()) & _capi.LC_DRAW_BAD_ROW:
        raise RuntimeError("sample() called with no probability mass")
    return int(tok.item())


def _prob_stats(probs) -> tuple[float, float]:
    """(-sum_{p>0} p ln p, max p) of one probability row on the device (lc_prob_stats)."""
    d = _dev.device()
    p = torch.as_tensor(np.asarray(probs, dtype=np.float64)).reshape(1, -1).to(d)
    out = torch.empty(2, dtype=torch.float64, device=d)
    V = p.shape[1]
    _capi.check(_capi.lib.lc_prob_stats(p.data_ptr(), V, 1, V, out[0:1].data_ptr(), out[1:2].data_ptr(),
                                        _dev.stream_ptr(d)), "lc_prob_stats")
    h, m = out.cpu().tolist()
    return h, m


def entropy(probs: np.ndarray) -> float:  # sampling.py:112-115
    return _prob_stats(probs)[0]


def max_prob(probs: np.ndarray) -> float:  # sampling.py:118-119
    return _prob_stats(probs)[1]


def hotspot_score(probs: np.ndarray, step: int, params: HotspotParams) -> float:
    if step < 0:
        raise ConfigError(f"step must be >= 0, got {step}")
    h, m = _prob_stats(probs)  # one launch for both (sampling.py:122-130)
    return h * (1.0 - m) / (1.0 + params.decay * step)


def select_hotspots(scores: np.ndarray, params: HotspotParams) -> tuple[int, ...]:
    """Min-max normalise, keep > threshold, cap by (-norm, t), ascending (sampling.py:135-145)."""
    scores = np.asarray(scores, dtype=np.float64)
    span = scores.max() - scores.min()
    if span == 0.0:
        return ()
    norm = (scores - scores.min()) / span
    pos = np.nonzero(norm > params.threshold)[0]
    if params.max_hotspots is not None and len(pos) > params.max_hotspots:
        pos = sorted(pos, key=lambda t: (-norm[t], t))[: params.max_hotspots]
    return tuple(sorted(int(t) for t in pos))


def row_scores(rows, temperature: float, decay: float, dev=None) -> np.ndarray:
    """Hotspot scores of a trajectory's rows: H(p) * (1 - max p) / (1 + decay*t)."""
    d = _dev.device(dev)
    z, dt = _rows_to_dev(rows, d)
    n, V = z.shape
    H = torch.empty(n, dtype=torch.float64, device=d)
    pm = torch.empty(n, dtype=torch.float64, device=d)
    _capi.check(_capi.lib.lc_row_entropy(z.data_ptr(), dt, V, V, n, float(temperature), H.data_ptr(),
                                         pm.data_ptr(), _dev.stream_ptr(d)), "lc_row_entropy")
    t = torch.arange(n, dtype=torch.float64, device=d)
    return (H * (1.0 - pm) / (1.0 + decay * t)).cpu().numpy()


def identify_hotspots(logits_seq, cfg: SamplingConfig, params: HotspotParams) -> tuple[int, ...]:
    if len(logits_seq) == 0:
        raise ConfigError("logits_seq must be non-empty")
    rows = logits_seq if isinstance(logits_seq, torch.Tensor) else np.stack([np.asarray(r) for r in logits_seq])
    return select_hotspots(row_scores(rows, cfg.temperature, params.decay), params)


# ---------------------------------------------------------------------- hot path


def make_tasks(row=None, temperature=1.0, top_k=None, top_p=1.0, draw_begin=None, draw_end=None, slot=None,
               pos=None, vocab=0, seed_base=0, u_index=-1, n=None) -> np.ndarray:
    """Host array of ``lc_task`` records (numpy structured, ABI layout)."""
    if n is None:
        for a in (row, slot, draw_begin):
            if a is not None and np.ndim(a) > 0:
                n = len(a)
                break
    t = np.zeros(n, dtype=_capi.TASK_DTYPE)
    t["row"] = -1 if row is None else row
    t["slot"] = -1 if slot is None else slot
    t["pos"] = 0 if pos is None else pos
    t["temperature"] = temperature
    t["top_k"] = 0 if top_k is None else top_k  # <= 0: none
    t["vocab"] = vocab
    t["top_p"] = top_p
    if draw_begin is None:
        draw_begin = np.arange(n)
        draw_end = draw_begin + 1
    t["draw_begin"] = draw_begin
    t["draw_end"] = draw_end
    t["seed_base"] = seed_base
    t["u_index"] = u_index
    return t


class Workspace:
    """Grow-only device scratch for the resample entry points."""

    def __init__(self, dev=None):
        self.dev = _dev.device(dev)
        self.buf = None

    def get(self, n_tasks: int, vocab: int) -> torch.Tensor:
        need = int(_capi.lib.lc_resample_workspace_bytes(n_tasks, vocab))
        if self.buf is None or self.buf.numel() < need:
            self.buf = torch.empty(need, dtype=torch.uint8, device=self.dev)
        return self.buf


_ws = {}


def _workspace(dev) -> Workspace:
    w = _ws.get(dev)
    if w is None:
        w = _ws[dev] = Workspace(dev)
    return w


def resample(rows: torch.Tensor, tasks, u: torch.Tensor | None = None, seeds: torch.Tensor | None = None,
             index: torch.Tensor | None = None, n_draws: int | None = None, counters: torch.Tensor | None = None,
             cache=None, out: tuple | None = None, kept: torch.Tensor | None = None,
             entropy: torch.Tensor | None = None, pmax: torch.Tensor | None = None):
    """Fused resample of device rows (or of cached rows when ``cache`` is given).

    ``tasks``: numpy TASK_DTYPE array or a uint8 device tensor of packed tasks.
    Draws come from ``u`` (fp64, one per draw) or from ``seeds`` (+ ``index``).
    Returns (tokens int32, flags uint8) device tensors, one entry per draw.
    ``kept`` (int32 device tensor, one per task, optional) receives each task's
    kept-set size K: truncate()'s kept ids are the first K of the row in
    (logit desc, id asc) order (sampling.py:71-94; V = untruncated, -1 = bad row).
    ``entropy`` / ``pmax`` (float64 device tensors, one per task, optional) receive the
    entropy and max probability of each task's row at its temperature (sampling.py:112-119),
    computed by an epilogue launch over the same rows.
    """
    dev = rows.device if rows is not None else cache.dev
    if isinstance(tasks, np.ndarray):
        n_tasks = len(tasks)
        if n_draws is None:
            n_draws = int(tasks["draw_end"].max()) if n_tasks else 0
        tt = torch.from_numpy(tasks.view(np.uint8).copy()).to(dev)
    else:
        tt = tasks
        n_tasks = tt.numel() // _capi.TASK_DTYPE.itemsize
        assert n_draws is not None
    if out is None:
        tok = torch.empty(max(n_draws, 1), dtype=torch.int32, device=dev)
        flags = torch.empty(max(n_draws, 1), dtype=torch.uint8, device=dev)
    else:
        tok, flags = out
    vocab = rows.shape[1] if rows is not None else cache.vocab
    ws = _workspace(dev).get(n_tasks, vocab)
    if kept is not None and (kept.dtype != torch.int32 or kept.numel() < n_tasks):
        raise ConfigError("kept must be an int32 tensor with one entry per task")
    for name, t in (("entropy", entropy), ("pmax", pmax)):
        if t is not None and (t.dtype != torch.float64 or t.numel() < n_tasks):
            raise ConfigError(f"{name} must be a float64 tensor with one entry per task")
    draws = _capi.LcDraws(_dev.ptr(u), _dev.ptr(seeds), _dev.ptr(index), tok.data_ptr(), _dev.ptr(flags),
                          _dev.ptr(kept), _dev.ptr(entropy), _dev.ptr(pmax))
    cnt = _dev.ptr(counters)
    if cache is None:
        if rows.dtype == torch.bfloat16:
            dt = _capi.LC_BF16
        elif rows.dtype == torch.float32:
            dt = _capi.LC_F32
        else:
            raise ConfigError(f"rows must be float32 or bfloat16, got {rows.dtype}")
        if rows.stride(1) != 1:
            raise ConfigError("rows must be row-major")
        rc = _capi.lib.lc_resample(rows.data_ptr(), dt, rows.shape[1], rows.stride(0), tt.data_ptr(), n_tasks, draws,
                                   ws.data_ptr(), ws.numel(), cnt, _dev.stream_ptr(dev))
    else:
        rc = _capi.lib.lc_cache_resample(cache.handle, tt.data_ptr(), n_tasks, draws, ws.data_ptr(), ws.numel(), cnt,
                                         _dev.stream_ptr(dev))
    _capi.check(rc, "lc_resample")
    return tok[:n_draws], flags[:n_draws]
