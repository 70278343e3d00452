"""Replay-aware generate on the device, for waves of requests.

Reference: ``InferenceEngine._generate`` (pkg/src/agentserve/engine.py:270-388)
over the synthetic model (model.py:31-83).  Per request:

1. ``key = StateKey.of(prompt)``; with STEP_WISE / HOTSPOT, ``lookup`` (a vocab
   mismatch is a miss, engine.py:286-289), pin;
2. replay the cached trajectory (step-wise: resample every position until the
   first divergent token; hotspot: resample hotspot positions only),
   engine.py:296-331;
3. the miss path: one "prefill" row for prompt + out, then decode rows until
   ``max_tokens`` tokens, each sampled with the request's RngStream
   (engine.py:336-347);
4. write back ``Z[:replayed] ++ new_rows`` under the key (engine.py:349-361).

Here a WAVE of requests with distinct keys runs each stage for every request
at once, entirely on the device:

* lookup / replay are ``LogitsCache.lookup_batch`` / ``replay_looked_up``;
* the write-back entry is allocated FIRST (``lc_cache_writeback``): its first
  ``replayed`` rows are the replayed prefix of the old entry, kept in place (an
  overwrite returns the old pages in page order) -- the ``np.concatenate`` copy
  of engine.py:353 disappears (f3);
* every decode step is one ``lc_engine_decode_step`` launch (fold the previous
  token into the digest, produce the next row straight into the write-back
  entry's slab row -- f1: no staging buffer, no insert copy -- and emit its
  resample task) plus one ``lc_cache_resample`` launch; the step loop has no
  host synchronisation; with ``LCB_ENGINE_GRAPH=1`` it is captured once per wave
  shape as a CUDA graph over engine-owned buffers and replayed by later waves of
  that shape (off by default: at 256-1024 requests per wave the eager loop is as
  fast, `profiles/r2_engine_graph_cache.jsonl`).

Semantics vs the reference's sequential calls: within a wave, all lookups happen
before all write-backs (in request order), and the looked-up entries stay pinned
until their own write-back.  When the logits budget does not evict during the
wave this is exactly the reference's call sequence for these requests (tokens,
replayed_len, diverged_at, the written entries: ``tests/test_gpu_engine.py``
against traces of the reference engine); under eviction pressure victims can
differ (other keys' entries are pinned a little longer).  The KV prefix trie,
forward-pass cost of prefill tokens and contribution profiling are outside this
path; the pass counters follow engine.py:364-371.
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _capi, _dev, mixing, sampling
from .errors import ConfigError
from .logits_cache import LogitsCache, ReplayOutcome, ReplayPolicy
from .sampling import HotspotParams, SamplingConfig


@dataclass(frozen=True)
class ModelConfig:
    """The synthetic next-token model (model.py:31-45)."""

    seed: int
    vocab_size: int = 256
    concentration: float = 2.0
    logit_range: float = 5.0

    def __post_init__(self):
        if self.vocab_size < 2:
            raise ConfigError(f"vocab_size must be >= 2, got {self.vocab_size}")
        if self.concentration < 0:
            raise ConfigError(f"concentration must be >= 0, got {self.concentration}")
        if self.logit_range <= 0:
            raise ConfigError(f"logit_range must be > 0, got {self.logit_range}")


@dataclass
class GenerateRequest:
    """engine.py:40-47."""

    agent_id: str
    prompt_tokens: list[int]
    sampling: SamplingConfig
    replay_policy: ReplayPolicy = ReplayPolicy.NONE
    request_id: str = ""
    hotspot: HotspotParams | None = None


@dataclass
class GenerateResult:
    """engine.py:50-63, without the KV-trie fields (prefill_tokens, matched_tokens)."""

    request_id: str
    agent_id: str
    tokens: list[int]
    outcome: ReplayOutcome
    was_revisit: bool
    prompt_len: int
    prefill_passes: int
    decode_passes: int
    prefill_input: int
    flags: list[int] = field(default_factory=list)


@dataclass
class CostReport:
    """Forward-pass meters (model.py:48-64) for the passes this path issues."""

    prefill_passes: int = 0
    decode_passes: int = 0


class WaveEngine:
    """``InferenceEngine.generate`` for waves of requests on one device (see module doc)."""

    def __init__(self, model: ModelConfig, logits_budget_bytes: int = 1 << 30,
                 hotspot_params: HotspotParams | None = None, *, dtype: str = "float32", max_tokens: int = 512,
                 key_capacity: int | None = None, page_rows: int | None = None, device=None):
        self.model = model
        self.dev = _dev.device(device)
        self.hotspot_params = hotspot_params or HotspotParams()
        self.cache = LogitsCache(logits_budget_bytes, vocab=model.vocab_size, dtype=dtype, max_rows=max_tokens,
                                 key_capacity=key_capacity, page_rows=page_rows, device=self.dev)
        self.dtype = dtype
        self.max_tokens = max_tokens
        self.cost = CostReport()
        self.agents: set[str] = set()
        self.generate_count = 0
        self._graphs = {}  # wave shape -> (captured decode loop, its buffers, its closure)
        self.request_log: list[GenerateResult] = []
        self.hotspot_flags: list[torch.Tensor] = []  # per hotspot wave: selection flags (lc_cache_hotspots)

    def register_agent(self, agent_id: str) -> None:
        self.agents.add(agent_id)

    def generate(self, request: GenerateRequest) -> GenerateResult:
        return self.generate_wave([request])[0]

    # ------------------------------------------------------------------------------------

    def _validate(self, requests):
        V = self.model.vocab_size
        if not requests:
            return
        pol = requests[0].replay_policy
        L = requests[0].sampling.max_tokens
        for q in requests:
            if q.agent_id not in self.agents:
                raise ConfigError(f"unknown agent {q.agent_id!r}")  # engine.py:273-274
            if not q.prompt_tokens:
                raise ConfigError("prompt must be non-empty")  # engine.py:258-259
            for t in q.prompt_tokens:
                if not (0 <= t < V):
                    raise ConfigError(f"token {t} outside vocabulary [0, {V})")  # engine.py:262-264
            if q.replay_policy is not pol:
                raise ConfigError("one replay policy per wave")
            if q.sampling.max_tokens != L:
                raise ConfigError("one max_tokens per wave")
        if L > self.max_tokens:
            raise ConfigError(f"max_tokens {L} exceeds the engine's {self.max_tokens}")

    def generate_wave(self, requests: list[GenerateRequest]) -> list[GenerateResult]:
        self._validate(requests)
        B = len(requests)
        if B == 0:
            return []
        if B > 65535:
            raise ConfigError("at most 65535 requests per wave")
        dev, V = self.dev, self.model.vocab_size
        L = requests[0].sampling.max_tokens
        policy = requests[0].replay_policy
        st = _dev.stream_ptr(dev)
        cfgs = [q.sampling for q in requests]
        seeds = _dev.u64_tensor([c.seed & mixing.MASK64 for c in cfgs], dev)
        T = torch.tensor([c.temperature for c in cfgs], dtype=torch.float64, device=dev)
        K = torch.tensor([c.top_k or 0 for c in cfgs], dtype=torch.int32, device=dev)
        P = torch.tensor([c.top_p for c in cfgs], dtype=torch.float64, device=dev)
        digests = mixing.hash_prompts([list(q.prompt_tokens) for q in requests], dev=dev)
        out = torch.zeros(B * L, dtype=torch.int32, device=dev)
        flags = torch.zeros(B * L, dtype=torch.uint8, device=dev)
        cache = self.cache if policy is not ReplayPolicy.NONE else None

        rep_h = np.zeros(B, dtype=np.int64)
        div_h = np.full(B, -1, dtype=np.int64)
        hit_h = np.zeros(B, dtype=bool)
        used_h = np.zeros(B, dtype=np.int64)
        if cache is not None:
            dig_h = _dev.u64_numpy(digests)
            if len(set(dig_h.tolist())) != B:
                raise ConfigError("the prompts of a wave must have distinct keys (run repeats in later waves)")
            slot, gen, ln, vv = cache.lookup_batch(digests)
            hit = (slot >= 0) & (vv == V)  # vocab mismatch is a miss (engine.py:288-289)
            slot_r = torch.where(hit, slot, torch.full_like(slot, -1))
            ln_r = torch.where(hit, torch.clamp(ln, max=L), torch.zeros_like(ln))
            _capi.check(_capi.lib.lc_cache_pin(cache.handle, slot_r.data_ptr(), gen.data_ptr(), B, 1, st),
                        "lc_cache_pin")  # engine.py:297
            draw_index = None
            if policy is ReplayPolicy.HOTSPOT:  # hotspots_for of every hit (engine.py:312), on the device
                draw_index = self._hotspot_draw_index(requests, slot_r, gen, L)
            tok, rep, div = cache.replay_looked_up(slot_r, gen, ln_r, vv, L, 1, seeds, T, K, P,
                                                   draw_index=draw_index)
            out.copy_(tok[: B * L])
            hit_h = hit.cpu().numpy()
            rep_h = rep[:B].cpu().numpy().astype(np.int64)
            div_h = div[:B].cpu().numpy().astype(np.int64)
            if policy is ReplayPolicy.HOTSPOT:  # draws consumed = hotspots replayed
                di = draw_index.view(B, L).cpu().numpy()
                used_h = ((di >= 0) & (np.arange(L)[None, :] < rep_h[:, None])).sum(1)
            else:
                used_h = rep_h.copy()
            rep_h[~hit_h] = 0
            div_h[~hit_h] = -1
            used_h[~hit_h] = 0
            # write-back entry first: rows [0, replayed) stay where they are (f3)
            keep = torch.from_numpy(rep_h.astype(np.int32)).to(dev)
            lens = torch.full((B,), L, dtype=torch.int32, device=dev)
            vocs = torch.full((B,), V, dtype=torch.int32, device=dev)
            wslot = torch.empty(B, dtype=torch.int32, device=dev)
            wgen = torch.empty(B, dtype=torch.int32, device=dev)
            _capi.check(_capi.lib.lc_cache_writeback(
                cache.handle, digests.data_ptr(), lens.data_ptr(), vocs.data_ptr(), keep.data_ptr(), gen.data_ptr(),
                B, None, _capi.LC_F32, 0, None, None, L, wslot.data_ptr(), wgen.data_ptr(), st),
                "lc_cache_writeback")
            cache._dirty()
            cache._stats()  # raises latched errors
            wlen = torch.empty(B, dtype=torch.int32, device=dev)
            _capi.check(_capi.lib.lc_cache_entry_len(cache.handle, wslot.data_ptr(), wgen.data_ptr(), B,
                                                     wlen.data_ptr(), st), "lc_cache_entry_len")
            staging = bool((wlen < 0).any().item())  # an entry evicted by its own write-back
        else:
            wslot = wgen = None
            staging = True

        # ---- miss path: prefill row + decode rows until max_tokens (engine.py:336-347)
        need = rep_h < L
        n_steps = int(L - rep_h[need].min()) if need.any() else 0
        if n_steps:
            temps = {c.temperature for c in cfgs}
            score_T = temps.pop() if (policy is ReplayPolicy.HOTSPOT and len(temps) == 1) else None
            self._decode(B, L, n_steps, rep_h, used_h, digests, out, flags, seeds, T, K, P, wslot, wgen, staging,
                         score_T)
        if cache is not None:
            pos = torch.arange(L, dtype=torch.int32, device=dev).repeat(B)
            s_rep, g_rep = wslot.repeat_interleave(L), wgen.repeat_interleave(L)  # (kept alive for the launch)
            _capi.check(_capi.lib.lc_cache_set_tokens(cache.handle, s_rep.data_ptr(), g_rep.data_ptr(),
                                                      pos.data_ptr(), out.data_ptr(), B * L, st),
                        "lc_cache_set_tokens")
            _capi.check(_capi.lib.lc_cache_pin(cache.handle, slot_r.data_ptr(), gen.data_ptr(), B, -1, st),
                        "lc_cache_pin")  # engine.py:331 (a no-op once overwritten)
            cache._dirty()
        toks = out.view(B, L).cpu().numpy()
        fl = flags.view(B, L).cpu().numpy()
        results = []
        for r, q in enumerate(requests):
            replayed = int(rep_h[r])
            if replayed < L:
                pre, dec, pin_ = 1, L - replayed - 1, len(q.prompt_tokens) + replayed
            else:
                pre, dec, pin_ = 0, 0, 0
            self.cost.prefill_passes += pre
            self.cost.decode_passes += dec
            oc = ReplayOutcome(replayed_len=replayed, diverged_at=int(div_h[r]) if div_h[r] >= 0 else None,
                               total_len=L, forward_passes_saved=(L - 1) - dec)
            res = GenerateResult(q.request_id, q.agent_id, toks[r].tolist(), oc, bool(hit_h[r]), len(q.prompt_tokens),
                                 pre, dec, pin_, fl[r].tolist())
            results.append(res)
            self.request_log.append(res)
        self.generate_count += B
        return results

    # ------------------------------------------------------------------------------------

    def _hotspot_draw_index(self, requests, slot_r, gen, L):
        """Device draw-index array [B * L] of the hits' hotspots, grouped by parameter set."""
        B = len(requests)
        di = torch.full((B * L,), -1, dtype=torch.int32, device=self.dev)
        groups = {}
        for r, q in enumerate(requests):
            hp = q.hotspot or self.hotspot_params
            groups.setdefault((q.sampling.temperature, hp), []).append(r)
        for (T, hp), rs in groups.items():
            idx = torch.tensor(rs, dtype=torch.int64, device=self.dev)
            d, _, fl = self.cache.hotspot_draw_index_device(slot_r[idx], gen[idx], L, T, hp)
            di.view(B, L)[idx] = d.view(len(rs), L)
            self.hotspot_flags.append(fl)
        return di

    def _decode(self, B, L, n_steps, rep_h, used_h, digests, out, flags, seeds, T, K, P, wslot, wgen, staging,
                score_T=None):
        dev = self.dev
        cache = self.cache if wslot is not None else None
        start = torch.from_numpy(rep_h.astype(np.int32)).to(dev)
        u0 = torch.from_numpy(used_h.astype(np.int64)).to(dev)
        io = dict(digests=digests, out=out, flags=flags, seeds=seeds, T=T, K=K, P=P, start=start, u0=u0)
        if cache is not None:
            io.update(wslot=wslot, wgen=wgen)
        if n_steps < 2 or os.environ.get("LCB_ENGINE_GRAPH", "0") != "1":
            self._decode_plan(B, L, n_steps, io, cache, staging, score_T)(_dev.stream_ptr(dev))
            return
        # The step loop has no host synchronisation: it is captured ONCE per wave shape into a CUDA
        # graph over engine-owned buffers, and each later wave of that shape copies its inputs in,
        # replays (one launch for fold + n_steps x (decode, resample)), and copies tokens / flags out.
        key = (B, L, n_steps, bool(staging), score_T, cache.epoch if cache is not None else None)
        ent = self._graphs.pop(key, None)
        if ent is None:
            bufs = {k: torch.empty_like(v) for k, v in io.items()}
            cur = torch.cuda.current_stream(dev)
            cs = torch.cuda.Stream(dev)
            cs.wait_stream(cur)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.stream(cs):
                run = self._decode_plan(B, L, n_steps, bufs, cache, staging, score_T, own_workspace=True)
                g.capture_begin(capture_error_mode="thread_local")
                try:
                    run(cs.cuda_stream)
                finally:
                    g.capture_end()
            cur.wait_stream(cs)
            ent = (g, bufs, run)
            while len(self._graphs) >= 8:
                self._graphs.pop(next(iter(self._graphs)))
        self._graphs[key] = ent  # (most recently used last)
        g, bufs, _ = ent
        for k, v in io.items():
            bufs[k].copy_(v, non_blocking=True)
        g.replay()
        out.copy_(bufs["out"], non_blocking=True)
        flags.copy_(bufs["flags"], non_blocking=True)

    def _decode_plan(self, B, L, n_steps, io, cache, staging, score_T, own_workspace=False):
        """The decode loop over the device buffers ``io`` as a function of the stream: the digest
        fold of prompt + replayed tokens, then per step one ``lc_engine_decode_step`` and one
        resample launch (+ the hotspot score epilogue).  Its scratch lives in the returned closure."""
        dev, V = self.dev, self.model.vocab_size
        start, u0, out, flags = io["start"], io["u0"], io["out"], io["flags"]
        dig = [torch.empty(B, dtype=torch.int64, device=dev), torch.empty(B, dtype=torch.int64, device=dev)]
        sdt = _capi.LC_F32 if self.dtype == "float32" else _capi.LC_BF16
        stg = None
        if staging:
            stg = torch.empty((B, V), dtype=torch.float32 if sdt == _capi.LC_F32 else torch.bfloat16, device=dev)
        tasks = torch.empty(B * _capi.TASK_DTYPE.itemsize, dtype=torch.uint8, device=dev)
        if own_workspace:  # (the shared workspace may be reallocated by later calls)
            ws = torch.empty(int(_capi.lib.lc_resample_workspace_bytes(B, V)), dtype=torch.uint8, device=dev)
        else:
            ws = sampling._workspace(dev).get(B, V)
        draws = _capi.LcDraws(None, io["seeds"].data_ptr(), None, out.data_ptr(), flags.data_ptr(), None, None, None)
        wslot = io.get("wslot")
        wgen = io.get("wgen")
        m = self.model
        steps = []
        for s in range(n_steps):
            a = _capi.LcDecodeStep(B, V, L, s, sdt, m.seed & mixing.MASK64, float(m.concentration),
                                   float(m.logit_range), start.data_ptr(), u0.data_ptr(), dig[s & 1].data_ptr(),
                                   dig[(s + 1) & 1].data_ptr(), out.data_ptr(),
                                   wslot.data_ptr() if cache is not None else None,
                                   wgen.data_ptr() if cache is not None else None,
                                   io["T"].data_ptr(), io["K"].data_ptr(), io["P"].data_ptr(),
                                   stg.data_ptr() if stg is not None else None, V, tasks.data_ptr())
            steps.append(a)
        pos_steps = None
        if score_T is not None and cache is not None:  # f2 epilogue: score each new row while it is in L2
            pos_steps = torch.empty((n_steps, B), dtype=torch.int32, device=dev)
            steps_ar = torch.arange(n_steps, dtype=torch.int32, device=dev)
        # (``cache is not None``, never ``if cache``: LogitsCache.__len__ reads the device counters)
        hnd = cache.handle if cache is not None else None
        digests = io["digests"]

        def run(st):
            # digest of prompt + out[:replayed] (engine.py:337: prefill of prompt + out)
            _capi.check(_capi.lib.lc_engine_fold(digests.data_ptr(), out.data_ptr(), L, start.data_ptr(), B,
                                                 dig[0].data_ptr(), st), "lc_engine_fold")
            if pos_steps is not None:  # (st is the current stream, eager or capturing)
                torch.add(start[None, :], steps_ar[:, None], out=pos_steps)
            for s_, a in enumerate(steps):
                _capi.check(_capi.lib.lc_engine_decode_step(hnd, C.byref(a), st), "lc_engine_decode_step")
                if stg is None:
                    rc = _capi.lib.lc_cache_resample(hnd, tasks.data_ptr(), B, draws, ws.data_ptr(), ws.numel(),
                                                     None, st)
                else:
                    rc = _capi.lib.lc_resample(stg.data_ptr(), sdt, V, V, tasks.data_ptr(), B, draws, ws.data_ptr(),
                                               ws.numel(), None, st)
                _capi.check(rc, "lc_resample")
                if pos_steps is not None:
                    _capi.check(_capi.lib.lc_cache_score_rows(hnd, wslot.data_ptr(), wgen.data_ptr(),
                                                              pos_steps[s_].data_ptr(), B, float(score_T), 0, st),
                                "lc_cache_score_rows")

        return run
