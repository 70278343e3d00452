"""HBM-resident logits cache behind the reference interface
(pkg/src/agentserve/logits_cache.py:1-183).

Names, arguments, semantics and error behaviour follow the reference:
``TOKEN_OVERHEAD_BYTES``, ``StateKey``, ``ReplayPolicy``, ``CachedTrajectory``,
``ReplayOutcome`` and ``LogitsCache`` with ``lookup`` / ``update`` / ``pin`` /
``unpin`` / ``hotspots_for`` / ``prefetch`` / ``drain_prefetch`` and the
attributes ``entries``, ``total_bytes``, ``budget_bytes``, ``lookups``,
``hits``, ``hotspot_computations``.  Storage, index and eviction are the CUDA
library (``lc_cache_*``): entries live in an HBM slab, lookups probe a GPU
hash table, and eviction is the reference's LRU-by-last-hit over accounted
bytes ``n*V*4 + 8*n``.

Deliberate differences:
* ``update`` copies the rows into HBM (the reference keeps a reference to the
  caller's float32 array, logits_cache.py:109); ``CachedTrajectory.logits_seq``
  is read back from the device on access;
* the slab width (vocabulary) is fixed when the device cache is created (the
  ``vocab`` argument, else the first update); narrower entries are stored
  as-is (and resampled over their own width), a wider or longer one rebuilds
  the device cache (live entries, pins, rounds and hotspot memos carried over;
  handles taken before the rebuild go stale);
* the slab holds ``page_capacity * page_rows`` rows: entries much narrower
  than the slab can make the accounted budget admit more rows than that, and
  such an insert raises ``CapacityError`` (rolled back) where the reference
  would store it.

Batched entry points (``lookup_batch``, ``insert_batch``, ``resample``,
``replay_stepwise``) take device tensors and never synchronise the host.
"""

from __future__ import annotations

import ctypes as C
from collections import deque
from dataclasses import dataclass, field
from enum import Enum

import numpy as np
import torch

from . import _capi, _dev, mixing, sampling
from .errors import CapacityError, ConfigError
from .sampling import HotspotParams, SamplingConfig

TOKEN_OVERHEAD_BYTES = 8  # logits_cache.py:23


@dataclass(frozen=True)
class StateKey:
    digest: int

    @classmethod
    def of(cls, prompt_tokens) -> "StateKey":
        return cls(mixing.hash_tokens(prompt_tokens))

    @classmethod
    def of_many(cls, prompts, dev=None) -> list["StateKey"]:
        return [cls(int(d)) for d in _dev.u64_numpy(mixing.hash_prompts(prompts, dev=dev))]


class ReplayPolicy(str, Enum):
    NONE = "none"
    STEP_WISE = "step_wise"
    HOTSPOT = "hotspot"


@dataclass
class ReplayOutcome:
    replayed_len: int
    diverged_at: int | None
    total_len: int
    forward_passes_saved: int

    @property
    def hit_ratio(self) -> float:
        if self.total_len == 0:
            return 0.0
        return self.replayed_len / self.total_len


class CachedTrajectory:
    """A (slot, generation) handle on a device-resident entry (logits_cache.py:41-56)."""

    def __init__(self, cache: "LogitsCache", slot: int, gen: int, n: int, vocab: int, digest: int,
                 created_round: int = 0):
        self._cache = cache
        self.slot = slot
        self.gen = gen
        self.epoch = cache._epoch  # device cache generation: a rebuild (``_grow``) makes the handle stale
        self._n = n
        self.vocab_size = vocab
        self.digest = digest
        self.created_round = created_round
        self.hotspots: dict[tuple, tuple[int, ...]] = {}
        self._logits = None
        self._tokens = None

    def __len__(self) -> int:
        return self._n

    def _positions(self):
        d = self._cache.dev
        s = torch.full((self._n,), self.slot, dtype=torch.int32, device=d)
        p = torch.arange(self._n, dtype=torch.int32, device=d)
        g = torch.full((self._n,), self.gen, dtype=torch.int64, device=d).to(torch.int32)
        return s, p, g

    def _check_live(self):
        if self.epoch != self._cache._epoch:
            raise ConfigError("stale CachedTrajectory: the device cache was rebuilt since it was looked up")

    @property
    def logits_seq(self) -> np.ndarray:
        if self._logits is None:
            self._logits = self.logits_device().cpu().numpy()
        return self._logits

    def logits_device(self) -> torch.Tensor:
        """The entry's rows as a float32 device tensor (zeros once the entry was overwritten
        or evicted: the read is checked against the handle's generation)."""
        self._check_live()
        return self._cache._gather(self.slot, self.gen, self._n, self.vocab_size)

    @property
    def token_seq(self) -> list[int]:
        if self._tokens is None:
            self._check_live()
            s, p, g = self._positions()
            out = torch.empty(self._n, dtype=torch.int32, device=self._cache.dev)
            if self._n:
                _capi.check(_capi.lib.lc_cache_tokens(self._cache.handle, s.data_ptr(), p.data_ptr(), g.data_ptr(),
                                                      self._n, out.data_ptr(), _dev.stream_ptr(self._cache.dev)),
                            "lc_cache_tokens")
            self._tokens = out.cpu().tolist()
        return self._tokens

    @property
    def nbytes(self) -> int:
        return self._n * self.vocab_size * 4 + TOKEN_OVERHEAD_BYTES * self._n

    def _meta(self, name):
        if self.epoch != self._cache._epoch:
            return None
        snap = self._cache._snapshot()
        if not snap["alive"][self.slot] or snap["gen"][self.slot] != self.gen:
            return None
        return snap[name][self.slot]

    @property
    def last_hit(self) -> int:
        v = self._meta("last_hit")
        return -1 if v is None else int(v)

    @property
    def pins(self) -> int:
        v = self._meta("pins")
        return 0 if v is None else int(v)


class LogitsCache:
    def __init__(self, budget_bytes: int = 1 << 30, *, vocab: int | None = None, dtype: str = "float32",
                 key_capacity: int | None = None, page_rows: int | None = None, max_rows: int = 1024,
                 page_capacity: int | None = None, device=None):
        if dtype not in ("float32", "bfloat16"):
            raise ConfigError(f"dtype must be float32 or bfloat16, got {dtype}")
        self.budget_bytes = int(budget_bytes)
        self.dev = _dev.device(device)
        self._dtype = dtype
        self._key_capacity = key_capacity
        self._page_rows = page_rows
        self._max_rows = max_rows
        self._page_capacity = page_capacity
        self.vocab = vocab
        self.handle = None
        self._prefetch_queue: deque = deque()
        self.hotspot_computations = 0
        self.hotspot_uncertain = 0  # selections with a decision inside the score bounds (reported)
        self._memo: dict[tuple[int, int], dict] = {}
        self._round: dict[tuple[int, int], int] = {}
        self._snap = None
        self._base = {"lookups": 0, "hits": 0, "hotspot_computations": 0}
        self._epoch = 0
        if vocab is not None:
            self._create(vocab)

    # -- device cache lifecycle ---------------------------------------------------------

    def _create(self, vocab: int):
        V = int(vocab)
        row_acct = V * 4 + TOKEN_OVERHEAD_BYTES
        budget_rows = self.budget_bytes // row_acct + 1
        page_rows = self._page_rows or (1 if self._max_rows <= 4 else 16)
        max_pages = -(-self._max_rows // page_rows)
        keys = self._key_capacity or max(int(min(65536, budget_rows + 64)), getattr(self, "_min_keys", 0))
        pages = self._page_capacity or int(budget_rows // page_rows + keys + 2 * max_pages + 8)
        cfg = _capi.LcCacheConfig(V, _capi.LC_F32 if self._dtype == "float32" else _capi.LC_BF16, page_rows,
                                  keys, pages, max_pages, self.dev.index or 0, self.budget_bytes)
        h = C.c_void_p()
        _capi.check(_capi.lib.lc_cache_create(C.byref(cfg), C.byref(h)), "lc_cache_create")
        self.handle = h
        self.epoch = getattr(self, "epoch", 0) + 1  # (a new device cache: captured launches are stale)
        self.vocab = V
        self.page_rows = page_rows
        self.max_pages = max_pages
        self.key_capacity = keys
        self.page_capacity = pages

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and _capi is not None and _capi.lib is not None:
            _capi.lib.lc_cache_destroy(h)
            self.handle = None

    def _stream(self):
        return _dev.stream_ptr(self.dev)

    def _stats(self):
        st = _capi.LcCacheStats()
        if self.handle is None:
            return st
        _capi.check(_capi.lib.lc_cache_stats_get(self.handle, C.byref(st), self._stream()), "lc_cache_stats_get")
        if st.error:
            code = int(st.error)
            if code == _capi.LC_E_CONFIG:
                raise ConfigError("entry wider than the slab or longer than max_rows")
            if code == _capi.LC_E_STATE:
                raise RuntimeError("write-back: the replayed prefix is no longer the key's live entry")
            raise CapacityError("logits cache slots/pages exhausted")
        return st

    def _snapshot(self):
        if self._snap is not None:
            return self._snap
        E = self.key_capacity
        d = self.dev
        out = {
            "digest": torch.empty(E, dtype=torch.int64, device=d),
            "last_hit": torch.empty(E, dtype=torch.int64, device=d),
            "gen": torch.empty(E, dtype=torch.int32, device=d),
            "pins": torch.empty(E, dtype=torch.int32, device=d),
            "nrows": torch.empty(E, dtype=torch.int32, device=d),
            "vocab": torch.empty(E, dtype=torch.int32, device=d),
            "alive": torch.empty(E, dtype=torch.uint8, device=d),
        }
        _capi.check(_capi.lib.lc_cache_snapshot(self.handle, *(out[k].data_ptr() for k in
                                                               ("digest", "last_hit", "gen", "pins", "nrows",
                                                                "vocab", "alive")), self._stream()),
                    "lc_cache_snapshot")
        snap = {k: v.cpu().numpy() for k, v in out.items()}
        snap["digest"] = snap["digest"].view(np.uint64)
        snap["gen"] = snap["gen"].view(np.uint32)
        self._snap = snap
        return snap

    def _dirty(self):
        self._snap = None

    # -- reference attributes -----------------------------------------------------------

    def __len__(self) -> int:
        return int(self._stats().entries) if self.handle is not None else 0

    @property
    def total_bytes(self) -> int:
        return int(self._stats().total_bytes) if self.handle is not None else 0

    @property
    def lookups(self) -> int:
        return self._base["lookups"] + (int(self._stats().lookups) if self.handle is not None else 0)

    @property
    def hits(self) -> int:
        return self._base["hits"] + (int(self._stats().hits) if self.handle is not None else 0)

    @property
    def entries(self) -> dict[int, CachedTrajectory]:
        if self.handle is None:
            return {}
        snap = self._snapshot()
        out = {}
        for s in np.flatnonzero(snap["alive"]):
            dg = int(snap["digest"][s])
            out[dg] = self._entry(int(s), int(snap["gen"][s]), int(snap["nrows"][s]), int(snap["vocab"][s]), dg)
        return out

    def _entry(self, slot, gen, n, vocab, digest):
        e = CachedTrajectory(self, slot, gen, n, vocab, digest, self._round.get((slot, gen), 0))
        e.hotspots = self._memo.setdefault((slot, gen), {})
        return e

    # -- batched device API ---------------------------------------------------------------

    def lookup_batch(self, digests: torch.Tensor):
        """digests: int64 device tensor of uint64 bit patterns.  Returns device tensors
        (slot, gen, len, vocab); slot -1 = miss.  Hits tick the clock in index order."""
        n = digests.numel()
        d = self.dev
        slot = torch.empty(n, dtype=torch.int32, device=d)
        gen = torch.empty(n, dtype=torch.int32, device=d)
        ln = torch.empty(n, dtype=torch.int32, device=d)
        vv = torch.empty(n, dtype=torch.int32, device=d)
        if self.handle is None:
            slot.fill_(-1)
            gen.zero_()
            ln.zero_()
            vv.zero_()
            self._base["lookups"] += n
            return slot, gen, ln, vv
        _capi.check(_capi.lib.lc_cache_lookup(self.handle, digests.data_ptr(), n, slot.data_ptr(), gen.data_ptr(),
                                              ln.data_ptr(), vv.data_ptr(), self._stream()), "lc_cache_lookup")
        self._dirty()
        return slot, gen, ln, vv

    def insert_batch(self, digests: torch.Tensor, lengths: torch.Tensor, vocabs: torch.Tensor, rows: torch.Tensor,
                     row_offsets: torch.Tensor, tokens: torch.Tensor, max_len: int):
        """Apply ``update`` for a batch in index order.  ``rows``: (total, stride)
        float32/bfloat16 device tensor; entry i is rows[row_offsets[i] + t]."""
        if self.handle is None:
            self._create(int(vocabs.max().item()) if vocabs.numel() else rows.shape[1])
        n = digests.numel()
        d = self.dev
        slot = torch.empty(n, dtype=torch.int32, device=d)
        gen = torch.empty(n, dtype=torch.int32, device=d)
        dt = _capi.LC_BF16 if rows.dtype == torch.bfloat16 else _capi.LC_F32
        if rows.dtype not in (torch.float32, torch.bfloat16):
            raise ConfigError(f"rows must be float32 or bfloat16, got {rows.dtype}")
        _capi.check(_capi.lib.lc_cache_insert(self.handle, digests.data_ptr(), lengths.data_ptr(), vocabs.data_ptr(),
                                              n, rows.data_ptr(), dt, rows.stride(0) if rows.dim() == 2 else 0,
                                              row_offsets.data_ptr(), _dev.ptr(tokens), int(max_len),
                                              slot.data_ptr(), gen.data_ptr(), self._stream()), "lc_cache_insert")
        self._dirty()
        return slot, gen

    def resample(self, tasks, **kw):
        """Fused resample of cached rows: tasks address rows by (slot, pos)."""
        return sampling.resample(None, tasks, cache=self, **kw)

    def replay_stepwise(self, digests: torch.Tensor, max_pos: int, n_branch: int, seeds: torch.Tensor,
                        temperature: torch.Tensor, top_k: torch.Tensor, top_p: torch.Tensor, counters=None,
                        bufs: dict | None = None, kept: torch.Tensor | None = None):
        """Lookup -> step-wise speculative resample of every cached position for
        n_branch branches per request -> acceptance (engine.py:285-331), all on
        the device.  Returns (tokens [n_req*max_pos*n_branch], replayed_len
        [n_req*n_branch], diverged_at, slot, len).  ``kept`` (int32 [n_req*max_pos],
        optional) receives each position's kept-set size (sampling.resample)."""
        slot, gen, ln, vv = self.lookup_batch(digests)
        tok, rep, div = self.replay_looked_up(slot, gen, ln, vv, max_pos, n_branch, seeds, temperature, top_k, top_p,
                                              counters=counters, bufs=bufs, kept=kept)
        return tok, rep, div, slot, ln

    def replay_looked_up(self, slot, gen, ln, vv, max_pos: int, n_branch: int, seeds: torch.Tensor,
                         temperature: torch.Tensor, top_k: torch.Tensor, top_p: torch.Tensor, counters=None,
                         bufs: dict | None = None, kept: torch.Tensor | None = None, draw_index=None,
                         hot_list=None):
        """The replay of ``replay_stepwise`` / ``replay_hotspot`` (``draw_index`` given) on
        lookup results the caller already holds (slot -1 = no replay; len capped at max_pos).
        Returns (tokens, replayed_len, diverged_at) device tensors."""
        n_req = slot.numel()
        b = self._replay_bufs(bufs, n_req, max_pos, n_branch)
        ntask = n_req * max_pos
        ndraw = ntask * n_branch
        st = self._stream()
        if draw_index is None:
            _capi.check(_capi.lib.lc_replay_tasks(slot.data_ptr(), ln.data_ptr(), vv.data_ptr(), n_req, max_pos,
                                                  n_branch, temperature.data_ptr(), top_k.data_ptr(),
                                                  top_p.data_ptr(), b["tasks"].data_ptr(), st), "lc_replay_tasks")
            ntask_run = ntask
        elif hot_list is not None:  # only the hotspot positions become tasks
            hp, hd = hot_list
            ntask_run = hp.numel()
            _capi.check(_capi.lib.lc_replay_tasks_hotspot_list(slot.data_ptr(), ln.data_ptr(), vv.data_ptr(),
                                                               hp.data_ptr(), hd.data_ptr(), ntask_run, max_pos,
                                                               n_branch, temperature.data_ptr(), top_k.data_ptr(),
                                                               top_p.data_ptr(), b["tasks"].data_ptr(), st),
                        "lc_replay_tasks_hotspot_list")
        else:
            _capi.check(_capi.lib.lc_replay_tasks_hotspot(slot.data_ptr(), ln.data_ptr(), vv.data_ptr(),
                                                          draw_index.data_ptr(), n_req, max_pos, n_branch,
                                                          temperature.data_ptr(), top_k.data_ptr(), top_p.data_ptr(),
                                                          b["tasks"].data_ptr(), st), "lc_replay_tasks_hotspot")
            ntask_run = ntask
        tok, flags = sampling.resample(None, b["tasks"][: ntask_run * _capi.TASK_DTYPE.itemsize], seeds=seeds,
                                       n_draws=ndraw, cache=self, counters=counters, out=(b["tok"], b["flags"]),
                                       kept=kept)
        self._cached_tokens(slot, gen, b, st)
        if draw_index is None:
            _capi.check(_capi.lib.lc_replay_accept(tok.data_ptr(), b["cached"].data_ptr(), ln.data_ptr(), n_req,
                                                   max_pos, n_branch, b["rep"].data_ptr(), b["div"].data_ptr(), st),
                        "lc_replay_accept")
        else:
            _capi.check(_capi.lib.lc_replay_accept_hotspot(tok.data_ptr(), b["cached"].data_ptr(), ln.data_ptr(),
                                                           draw_index.data_ptr(), n_req, max_pos, n_branch,
                                                           b["rep"].data_ptr(), b["div"].data_ptr(), st),
                        "lc_replay_accept_hotspot")
        return tok, b["rep"], b["div"]

    def replay_windowed(self, slot, gen, ln, vv, max_pos: int, n_branch: int, seeds: torch.Tensor,
                        temperature: torch.Tensor, top_k: torch.Tensor, top_p: torch.Tensor, window: int = 8,
                        counters=None, bufs: dict | None = None):
        """Step-wise replay (engine.py:296-331) evaluated ``window`` positions at a time on
        lookup results: a request's rows are resampled only while one of its branches is still
        replaying.  Same (tokens at accepted positions, replayed_len, diverged_at) as
        ``replay_looked_up`` with no ``draw_index``; rows past every branch's divergence are
        never read.  One small host read per window (the live-branch count) decides whether
        the next window runs.  Returns (tokens, replayed_len, diverged_at, windows run)."""
        n_req = slot.numel()
        b = self._replay_bufs(bufs, n_req, max_pos, n_branch)
        W = max(1, min(int(window), max_pos))
        st = self._stream()
        d = self.dev
        if b.get("wshape") != (n_req, W):
            b["wshape"] = (n_req, W)
            b["wtasks"] = torch.empty(max(n_req * W, 1) * _capi.TASK_DTYPE.itemsize, dtype=torch.uint8, device=d)
            b["live"] = torch.empty(max(n_req, 1), dtype=torch.int32, device=d)
            b["nlive"] = torch.zeros(1, dtype=torch.int32, device=d)
            b["nlive_h"] = torch.zeros(1, dtype=torch.int32, pin_memory=True)
        ndraw = n_req * max_pos * n_branch
        _capi.check(_capi.lib.lc_replay_window_init(ln.data_ptr(), n_req, max_pos, n_branch, b["rep"].data_ptr(),
                                                    b["div"].data_ptr(), b["live"].data_ptr(), b["nlive"].data_ptr(),
                                                    st), "lc_replay_window_init")
        self._cached_tokens(slot, gen, b, st)
        windows = 0
        for w0 in range(0, max_pos, W):
            _capi.check(_capi.lib.lc_replay_window_tasks(slot.data_ptr(), ln.data_ptr(), vv.data_ptr(),
                                                         b["live"].data_ptr(), n_req, max_pos, n_branch, w0, W,
                                                         temperature.data_ptr(), top_k.data_ptr(), top_p.data_ptr(),
                                                         b["wtasks"].data_ptr(), st), "lc_replay_window_tasks")
            sampling.resample(None, b["wtasks"], seeds=seeds, n_draws=ndraw, cache=self, counters=counters,
                              out=(b["tok"], b["flags"]))
            _capi.check(_capi.lib.lc_replay_window_accept(b["tok"].data_ptr(), b["cached"].data_ptr(), ln.data_ptr(),
                                                          n_req, max_pos, n_branch, w0, W, b["rep"].data_ptr(),
                                                          b["div"].data_ptr(), b["live"].data_ptr(),
                                                          b["nlive"].data_ptr(), st), "lc_replay_window_accept")
            windows += 1
            b["nlive_h"].copy_(b["nlive"], non_blocking=True)  # (st is torch's current stream)
            torch.cuda.current_stream(d).synchronize()
            if int(b["nlive_h"][0]) == 0:
                break
        return b["tok"], b["rep"], b["div"], windows

    def _replay_bufs(self, bufs, n_req: int, max_pos: int, n_branch: int) -> dict:
        """Device buffers of a replay call, reused across calls of the same shape (a
        caller's ``bufs`` dict is rebuilt whenever (n_req, max_pos, n_branch) changes)."""
        b = bufs if bufs is not None else {}
        shape = (n_req, max_pos, n_branch)
        if b.get("shape") != shape:
            d = self.dev
            ntask = n_req * max_pos
            ndraw = ntask * n_branch
            b.clear()
            b["shape"] = shape
            b["tasks"] = torch.empty(ntask * _capi.TASK_DTYPE.itemsize, dtype=torch.uint8, device=d)
            b["tok"] = torch.empty(max(ndraw, 1), dtype=torch.int32, device=d)
            b["flags"] = torch.empty(max(ndraw, 1), dtype=torch.uint8, device=d)
            b["cached"] = torch.empty(max(ntask, 1), dtype=torch.int32, device=d)
            b["pos"] = torch.arange(max_pos, dtype=torch.int32, device=d).repeat(n_req)
            b["rep"] = torch.empty(max(n_req * n_branch, 1), dtype=torch.int32, device=d)
            b["div"] = torch.empty(max(n_req * n_branch, 1), dtype=torch.int32, device=d)
        return b

    def _cached_tokens(self, slot, gen, b, st):
        """b["cached"][r * max_pos + t] = the looked-up entry's token t (-1 past its end)."""
        n_req, max_pos, _ = b["shape"]
        ntask = n_req * max_pos
        slots_rep = slot.repeat_interleave(max_pos)
        gens_rep = gen.repeat_interleave(max_pos)
        _capi.check(_capi.lib.lc_cache_tokens(self.handle, slots_rep.data_ptr(), b["pos"].data_ptr(),
                                              gens_rep.data_ptr(), ntask, b["cached"].data_ptr(), st),
                    "lc_cache_tokens")

    @staticmethod
    def hotspot_draw_index(hotspots, max_pos: int, dev=None) -> torch.Tensor:
        """Device array [n_req * max_pos]: the RngStream draw number of each hotspot position
        (hotspots of the request before it), -1 elsewhere -- the layout replay_hotspot takes."""
        di = np.full((len(hotspots), max_pos), -1, dtype=np.int32)
        for r, hs in enumerate(hotspots):
            hs = sorted(t for t in hs if 0 <= t < max_pos)
            di[r, hs] = np.arange(len(hs), dtype=np.int32)
        return torch.from_numpy(di.reshape(-1)).to(_dev.device(dev))

    @staticmethod
    def hotspot_list(draw_index: torch.Tensor):
        """Compact (flat position, draw number) lists of the hotspots in a draw-index array."""
        pos = torch.nonzero(draw_index >= 0).flatten()
        return pos.to(torch.int64), draw_index[pos].to(torch.int32).contiguous()

    def replay_hotspot(self, digests: torch.Tensor, max_pos: int, n_branch: int, seeds: torch.Tensor,
                       temperature: torch.Tensor, top_k: torch.Tensor, top_p: torch.Tensor, hotspots=None,
                       counters=None, bufs: dict | None = None, draw_index: torch.Tensor | None = None,
                       hot_list=None, kept: torch.Tensor | None = None):
        """ReplayPolicy.HOTSPOT for a batch (engine.py:311-326): request r samples only at
        the positions in ``hotspots[r]`` (RngStream draw number = hotspots before t) and
        copies the cached token elsewhere; the replay stops after the first hotspot sample
        that differs from the cache.  Same returns as ``replay_stepwise``; the token array
        holds the engine's ``out`` tokens at every replayed position."""
        n_req = digests.numel()
        if draw_index is None:
            if hotspots is None or len(hotspots) != n_req:
                raise ConfigError("one hotspot tuple per request")
            draw_index = self.hotspot_draw_index(hotspots, max_pos, self.dev)
        elif draw_index.numel() != n_req * max_pos:
            raise ConfigError("draw_index must hold n_req * max_pos entries")
        slot, gen, ln, vv = self.lookup_batch(digests)
        tok, rep, div = self.replay_looked_up(slot, gen, ln, vv, max_pos, n_branch, seeds, temperature, top_k, top_p,
                                              counters=counters, bufs=bufs, kept=kept, draw_index=draw_index,
                                              hot_list=hot_list)
        return tok, rep, div, slot, ln

    # -- reference API --------------------------------------------------------------------

    def lookup(self, key: StateKey) -> CachedTrajectory | None:
        dg = _dev.u64_tensor([key.digest], self.dev)
        slot, gen, ln, vv = self.lookup_batch(dg)
        s = int(slot.item())
        if s < 0:
            return None
        return self._entry(s, int(gen.view(torch.int32).item()) & 0xFFFFFFFF, int(ln.item()), int(vv.item()),
                           key.digest)

    def update(self, key: StateKey, logits_seq, token_seq, round_index: int = 0,
               prefetch_config: tuple[SamplingConfig, HotspotParams] | None = None) -> CachedTrajectory:
        if isinstance(logits_seq, torch.Tensor):
            z = logits_seq
            if z.dtype not in (torch.float32, torch.bfloat16):
                z = z.to(torch.float32)
        else:
            z = torch.from_numpy(np.ascontiguousarray(np.asarray(logits_seq, dtype=np.float32)))
        tokens = list(token_seq)
        if z.dim() != 2 or z.shape[0] != len(tokens):  # logits_cache.py:110-113
            raise ConfigError(f"logits/token length mismatch: {tuple(z.shape)} vs {len(tokens)}")
        n, V = z.shape
        if self.handle is None:
            self._max_rows = max(self._max_rows, n)
            self._create(max(V, self.vocab or 0))
        elif V > self.vocab or n > self._max_rows:
            self._rebuild(max(V, self.vocab), max(n, self._max_rows))
        z = z.to(self.dev).contiguous()
        if n == 0:
            z = torch.zeros((1, V), dtype=z.dtype, device=self.dev)
        d = self.dev
        dg = _dev.u64_tensor([key.digest], d)
        slot, gen = self.insert_batch(
            dg, torch.tensor([n], dtype=torch.int32, device=d), torch.tensor([V], dtype=torch.int32, device=d), z,
            torch.zeros(1, dtype=torch.int64, device=d),
            torch.tensor(tokens if tokens else [0], dtype=torch.int32, device=d), n)
        self._stats()  # raises latched errors
        s, g = int(slot.item()), int(gen.item()) & 0xFFFFFFFF
        self._round[(s, g)] = round_index
        self._memo[(s, g)] = {}
        entry = self._entry(s, g, n, V, key.digest)
        if prefetch_config is not None:
            self._prefetch_queue.append((key.digest, *prefetch_config))
        return entry

    def _rebuild(self, V: int, max_rows: int):
        """Rebuild the device cache wider and/or longer (an entry wider than the slab or
        longer than ``max_rows`` arrived).  Live entries are re-inserted in LRU order, so
        their relative last-hit order -- hence every later victim choice -- is kept, with
        their pins, rounds and hotspot memos; handles taken before go stale (epoch)."""
        snap = self._snapshot()
        live = sorted((int(s) for s in np.flatnonzero(snap["alive"])), key=lambda s: int(snap["last_hit"][s]))
        saved = []
        for s in live:
            g, n, v, dg = int(snap["gen"][s]), int(snap["nrows"][s]), int(snap["vocab"][s]), int(snap["digest"][s])
            toks = self._entry(s, g, n, v, dg).token_seq
            saved.append((dg, self._gather(s, g, n, v), toks, int(snap["pins"][s]), self._round.get((s, g), 0),
                          self._memo.get((s, g), {})))
        st = self._stats()
        self._base["lookups"] += int(st.lookups)
        self._base["hits"] += int(st.hits)
        _capi.lib.lc_cache_destroy(self.handle)
        self.handle = None
        self._memo = {}
        self._round = {}
        self._epoch += 1
        self._max_rows = max_rows
        self._min_keys = len(saved) + 64
        self._create(V)
        for dg, rows, toks, pins, rnd, memo in saved:
            e = self.update(StateKey(dg), rows, toks, round_index=rnd)
            self._memo[(e.slot, e.gen)] = memo
            for _ in range(pins):
                self._pin(e, 1)

    def _gather(self, slot: int, gen: int, n: int, vocab: int) -> torch.Tensor:
        d = self.dev
        out = torch.empty((max(n, 0), vocab), dtype=torch.float32, device=d)
        if n:
            s = torch.full((n,), slot, dtype=torch.int32, device=d)
            p = torch.arange(n, dtype=torch.int32, device=d)
            g = torch.full((n,), gen, dtype=torch.int64, device=d).to(torch.int32)
            _capi.check(_capi.lib.lc_cache_gather(self.handle, s.data_ptr(), p.data_ptr(), g.data_ptr(), n,
                                                  out.data_ptr(), _capi.LC_F32, vocab, self._stream()),
                        "lc_cache_gather")
        return out

    def _pin(self, entry: CachedTrajectory, delta: int):
        d = self.dev
        s = torch.tensor([entry.slot], dtype=torch.int32, device=d)
        g = torch.tensor([entry.gen], dtype=torch.int64, device=d).to(torch.int32)
        _capi.check(_capi.lib.lc_cache_pin(self.handle, s.data_ptr(), g.data_ptr(), 1, delta, self._stream()),
                    "lc_cache_pin")
        self._dirty()

    def pin(self, entry: CachedTrajectory) -> None:
        self._pin(entry, 1)

    def unpin(self, entry: CachedTrajectory) -> None:
        self._pin(entry, -1)

    # -- hotspot precomputation (logits_cache.py:153-183) --------------------------------

    def row_scores(self, entry: CachedTrajectory, temperature: float, decay: float) -> np.ndarray:
        """sampling.row_scores of the entry's rows, read from the slab in place
        (lc_cache_row_entropy: no gather of the rows)."""
        n = len(entry)
        d = self.dev
        entry._check_live()
        s, p, g = entry._positions()
        H = torch.empty(n, dtype=torch.float64, device=d)
        pm = torch.empty(n, dtype=torch.float64, device=d)
        _capi.check(_capi.lib.lc_cache_row_entropy(self.handle, s.data_ptr(), p.data_ptr(), g.data_ptr(), n,
                                                   float(temperature), H.data_ptr(), pm.data_ptr(), self._stream()),
                    "lc_cache_row_entropy")
        t = torch.arange(n, dtype=torch.float64, device=d)
        return (H * (1.0 - pm) / (1.0 + decay * t)).cpu().numpy()

    def score_rows(self, slot: torch.Tensor, gen: torch.Tensor, temperature: float, max_len: int | None = None):
        """Hotspot scores of every row of the entries (slot, gen) at ``temperature``, kept
        beside the rows in the slab (lc_cache_score_rows; rows already scored at this T
        are skipped)."""
        n = slot.numel()
        L = int(max_len or self.max_pages * self.page_rows)
        if n == 0 or L == 0:
            return
        s_rep = slot.to(torch.int32).repeat_interleave(L)
        g_rep = gen.to(torch.int32).repeat_interleave(L)
        pos = torch.arange(L, dtype=torch.int32, device=self.dev).repeat(n)
        _capi.check(_capi.lib.lc_cache_score_rows(self.handle, s_rep.data_ptr(), g_rep.data_ptr(), pos.data_ptr(),
                                                  n * L, float(temperature), 1, self._stream()),
                    "lc_cache_score_rows")

    def hotspot_draw_index_device(self, slot: torch.Tensor, gen: torch.Tensor, max_pos: int, temperature: float,
                                  params: HotspotParams, score: bool = True):
        """Hotspots of n entries selected on the device (select_hotspots over the entries'
        scores, sampling.py:133-160) in the replay's draw-index layout: [n * max_pos] int32,
        the draw number of hotspot t (= hotspots before t), -1 elsewhere (dead or missing
        entries: none).  Returns (draw_index, n_hot, flags) device tensors; flags bit 0 = a
        decision the score bounds cannot certify against the reference."""
        n = slot.numel()
        d = self.dev
        di = torch.full((max(n * max_pos, 1),), -1, dtype=torch.int32, device=d)
        nh = torch.zeros(max(n, 1), dtype=torch.int32, device=d)
        fl = torch.zeros(max(n, 1), dtype=torch.uint8, device=d)
        if n == 0:
            return di[:0], nh[:0], fl[:0]
        s32, g32 = slot.to(torch.int32).contiguous(), gen.to(torch.int32).contiguous()
        if score:
            self.score_rows(s32, g32, temperature)
        mh = -1 if params.max_hotspots is None else int(params.max_hotspots)
        _capi.check(_capi.lib.lc_cache_hotspots(self.handle, s32.data_ptr(), g32.data_ptr(), n, int(max_pos),
                                                float(temperature), float(params.decay), float(params.threshold), mh,
                                                di.data_ptr(), nh.data_ptr(), fl.data_ptr(), self._stream()),
                    "lc_cache_hotspots")
        return di[: n * max_pos], nh[:n], fl[:n]

    def hotspots_for(self, entry: CachedTrajectory, cfg: SamplingConfig, params: HotspotParams) -> tuple[int, ...]:
        """logits_cache.py:153-163: memoised per entry and parameter set; computed on the
        device from the scores kept beside the rows (no row leaves the slab)."""
        key = params.cache_key(cfg.temperature)
        cached = entry.hotspots.get(key)
        if cached is None:
            if len(entry) == 0:
                raise ConfigError("logits_seq must be non-empty")
            entry._check_live()
            n = len(entry)
            s = torch.tensor([entry.slot], dtype=torch.int32, device=self.dev)
            g = torch.tensor([entry.gen], dtype=torch.int64, device=self.dev).to(torch.int32)
            di, nh, fl = self.hotspot_draw_index_device(s, g, n, cfg.temperature, params)
            fl_h = int(fl.item())
            if fl_h & 4:
                raise ConfigError("stale CachedTrajectory: the entry was overwritten or evicted")
            if fl_h & 1:
                self.hotspot_uncertain += 1
            cached = tuple(int(t) for t in torch.nonzero(di >= 0).flatten().cpu().tolist())
            entry.hotspots[key] = cached
            self.hotspot_computations += 1
        return cached

    def prefetch(self, key: StateKey, cfg: SamplingConfig, params: HotspotParams) -> None:
        if self.handle is None:
            return
        snap = self._snapshot()
        hit = np.flatnonzero(snap["alive"].astype(bool) & (snap["digest"] == np.uint64(key.digest)))
        if len(hit) == 0:
            return
        s = int(hit[0])
        e = self._entry(s, int(snap["gen"][s]), int(snap["nrows"][s]), int(snap["vocab"][s]), key.digest)
        self.hotspots_for(e, cfg, params)

    def drain_prefetch(self, limit: int | None = None) -> int:
        ran = 0
        while self._prefetch_queue and (limit is None or ran < limit):
            digest, cfg, params = self._prefetch_queue.popleft()
            self.prefetch(StateKey(digest), cfg, params)
            ran += 1
        return ran
