"""The wave engine (paper_2604_17353_b200.engine) against traces of
the REFERENCE engine (tests/golden/engine_traces.json, made by make_engine_golden.py from
agentserve.engine.InferenceEngine): tokens, ReplayOutcome, pass counters and the
written-back cache entries (length, tokens, SHA-1 of the float32 rows) bit-exact.
Plus the write-back mechanics: the replayed prefix stays in its pages (no copy), the
producer writes the new rows straight into the slab, a dead write-back falls back to
staging rows."""

from __future__ import annotations

import ctypes as C
import hashlib

import numpy as np
import pytest
import torch

from oracle import mixing_ref, sampling_ref
from tests.golden_io import load_json

pytestmark = pytest.mark.gpu

lcb = pytest.importorskip("paper_2604_17353_b200")
from paper_2604_17353_b200 import _capi, _dev  # noqa: E402
from paper_2604_17353_b200.engine import GenerateRequest, ModelConfig, WaveEngine  # noqa: E402

DEV = torch.device("cuda", 0)
TRACES = load_json("engine_traces.json")
POL = {"step_wise": lcb.ReplayPolicy.STEP_WISE, "hotspot": lcb.ReplayPolicy.HOTSPOT, "none": lcb.ReplayPolicy.NONE}


def _engine(sc, **kw):
    seed, V, conc, rng = sc["model"]
    hp = lcb.HotspotParams(*sc["hp"]) if sc.get("hp") else lcb.HotspotParams()
    Lmax = max(sc["L"]) if isinstance(sc["L"], list) else sc["L"]
    eng = WaveEngine(ModelConfig(seed=seed, vocab_size=V, concentration=conc, logit_range=rng), 1 << 30, hp,
                     max_tokens=Lmax, device=DEV, **kw)
    eng.register_agent("a")
    return eng


@pytest.mark.parametrize("graph", ["1", "0"])
@pytest.mark.parametrize("name", [sc["name"] for sc in TRACES])
def test_wave_engine_matches_reference_engine(name, graph, monkeypatch):
    # graph "1": the decode loop runs as one CUDA graph per wave (default); "0": eager launches
    monkeypatch.setenv("LCB_ENGINE_GRAPH", graph)
    sc = next(s for s in TRACES if s["name"] == name)
    eng = _engine(sc)
    for w, wave in enumerate(sc["waves"]):
        reqs = [GenerateRequest("a", pr, lcb.SamplingConfig(temperature=sc["T"], top_k=sc["k"], top_p=sc["p"],
                                                            max_tokens=r["max_tokens"], seed=r["seed"]),
                                POL[sc["policy"]], request_id=f"w{w}r{i}")
                for i, (pr, r) in enumerate(zip(sc["prompts"], wave))]
        got = eng.generate_wave(reqs)
        for i, (g, r) in enumerate(zip(got, wave)):
            where = (name, w, i)
            assert g.tokens == r["tokens"], where
            assert g.outcome.replayed_len == r["replayed_len"], where
            assert g.outcome.diverged_at == r["diverged_at"], where
            assert g.outcome.total_len == r["total_len"], where
            assert g.outcome.forward_passes_saved == r["forward_passes_saved"], where
            assert g.was_revisit == r["was_revisit"], where
            assert (g.prefill_passes, g.decode_passes, g.prefill_input) == (
                r["prefill_passes"], r["decode_passes"], r["prefill_input"]), where
            assert not any(f & (_capi.LC_DRAW_UNRESOLVED | _capi.LC_DRAW_BAD_ROW) for f in g.flags), where
    cache = eng.cache
    assert cache.total_bytes == sc["total_bytes"]
    assert (cache.lookups, cache.hits) == (sc["lookups"], sc["hits"])
    ents = cache.entries
    assert sorted(str(d) for d in ents) == sorted(sc["entries"])
    for d, e in ents.items():
        want = sc["entries"][str(d)]
        assert len(e) == want["n"] and e.token_seq == want["tokens"], d
        rows = np.ascontiguousarray(e.logits_seq, dtype=np.float32)
        assert hashlib.sha1(rows.tobytes()).hexdigest() == want["sha1"], d


def _page_table(cache, slot):
    """Entry ``slot``'s page table (a device array of the handle), copied to the host."""
    pages, maxp, pr = C.c_void_p(), C.c_int32(), C.c_int32()
    _capi.check(_capi.lib.lc_cache_page_table(cache.handle, C.byref(pages), C.byref(maxp), C.byref(pr)))
    torch.cuda.synchronize(DEV)
    n = cache.key_capacity * maxp.value
    host = (C.c_int32 * n)()
    cudart = C.CDLL("libcudart.so.12")  # already loaded by liblcb200.so
    assert cudart.cudaMemcpy(host, pages, C.c_size_t(n * 4), C.c_int(2)) == 0  # device -> host
    return np.frombuffer(host, dtype=np.int32).reshape(cache.key_capacity, maxp.value)[slot].copy()


def test_writeback_keeps_replayed_prefix_in_place():
    """hit -> diverge at t -> write-back -> lookup: rows [0, replayed) keep their slab pages
    (an overwrite returns the old pages in page order), the decoded rows are the producer's
    rows for prompt + out, and the entry is the reference's merged trajectory."""
    V, L = 512, 40
    eng = WaveEngine(ModelConfig(seed=4, vocab_size=V), 1 << 30, max_tokens=L, page_rows=8, device=DEV)
    eng.register_agent("a")
    prompt = [5, 6, 7, 8]
    Tw = 0.5
    cfg = lambda s: lcb.SamplingConfig(temperature=Tw, top_p=1.0, max_tokens=L, seed=s)  # noqa: E731
    r1 = eng.generate(GenerateRequest("a", prompt, cfg(1), lcb.ReplayPolicy.STEP_WISE))
    e1 = eng.cache.lookup(lcb.StateKey.of(prompt))
    pages1 = _page_table(eng.cache, e1.slot).copy()
    rows1 = e1.logits_seq.copy()
    # find a seed whose replay diverges in the middle
    for s in range(2, 200):
        r2 = eng.generate(GenerateRequest("a", prompt, cfg(s), lcb.ReplayPolicy.STEP_WISE))
        if 8 < r2.outcome.replayed_len < L:
            break
        rows1 = eng.cache.lookup(lcb.StateKey.of(prompt)).logits_seq.copy()
        pages1 = _page_table(eng.cache, e1.slot).copy()
    rep = r2.outcome.replayed_len
    assert 8 < rep < L and r2.outcome.diverged_at == rep - 1
    e2 = eng.cache.lookup(lcb.StateKey.of(prompt))
    assert e2.slot == e1.slot
    pages2 = _page_table(eng.cache, e2.slot)
    kp = -(-rep // 8)
    assert np.array_equal(pages2[:kp], pages1[:kp])  # the replayed prefix did not move
    rows2 = e2.logits_seq
    assert np.array_equal(rows2[:rep], rows1[:rep])
    # new rows: the reference producer at prompt + out[:t]
    for t in range(rep, L):
        st = mixing_ref.mix2(4, mixing_ref.hash_tokens(prompt + r2.tokens[:t]))
        assert np.array_equal(rows2[t], mixing_ref.fill_rows_np([st], V, 2.0)[0]), t
    assert e2.token_seq == r2.tokens
    # and the tokens are the reference engine's: sample(truncate(softmax)) with RngStream(seed)
    for t in range(L):
        q = sampling_ref.truncate(sampling_ref.softmax(rows2[t], Tw), None, 1.0)
        assert sampling_ref.draw(q, mixing_ref.uniform(s, t)) == r2.tokens[t], t


def test_dead_writeback_entry_uses_staging_rows():
    """A budget of one entry: the wave's second write-back evicts the first one (its new
    entry is the LRU end once the old pinned entry is overwritten), so that request's
    decode samples staging rows; tokens equal a cold engine's."""
    V, L = 256, 12
    row = V * 4 + 8
    eng = WaveEngine(ModelConfig(seed=8, vocab_size=V), row * L + 16, max_tokens=L, device=DEV)
    eng.register_agent("a")
    p1, p2 = [1, 2, 3], [4, 5, 6]
    c = lambda s: lcb.SamplingConfig(temperature=1.0, max_tokens=L, seed=s)  # noqa: E731
    eng.generate(GenerateRequest("a", p1, c(1), lcb.ReplayPolicy.STEP_WISE))
    res = eng.generate_wave([GenerateRequest("a", p1, c(2), lcb.ReplayPolicy.STEP_WISE),
                             GenerateRequest("a", p2, c(3), lcb.ReplayPolicy.STEP_WISE)])
    cold = WaveEngine(ModelConfig(seed=8, vocab_size=V), 1 << 30, max_tokens=L, device=DEV)
    cold.register_agent("a")
    ref = cold.generate_wave([GenerateRequest("a", p1, c(2), lcb.ReplayPolicy.NONE),
                              GenerateRequest("a", p2, c(3), lcb.ReplayPolicy.NONE)])
    assert [r.tokens for r in res] == [r.tokens for r in ref]  # step-wise tokens never depend on the cache
    assert res[0].was_revisit and not res[1].was_revisit


def test_wave_rejects_duplicate_keys_and_mixed_policies():
    eng = WaveEngine(ModelConfig(seed=1, vocab_size=64), max_tokens=8, device=DEV)
    eng.register_agent("a")
    c = lcb.SamplingConfig(max_tokens=8)
    with pytest.raises(lcb.ConfigError):
        eng.generate_wave([GenerateRequest("a", [1, 2], c, lcb.ReplayPolicy.STEP_WISE)] * 2)
    with pytest.raises(lcb.ConfigError):
        eng.generate_wave([GenerateRequest("a", [1, 2], c, lcb.ReplayPolicy.STEP_WISE),
                           GenerateRequest("a", [1, 3], c, lcb.ReplayPolicy.NONE)])
    with pytest.raises(lcb.ConfigError):
        eng.generate(GenerateRequest("b", [1], c))
    with pytest.raises(lcb.ConfigError):
        eng.generate(GenerateRequest("a", [64], c))


def test_decode_graph_reuse_equals_eager(monkeypatch):
    """Waves of one shape replay the captured decode loop (one graph per shape) and give the
    eager loop's tokens, outcomes and cache entries."""
    model = ModelConfig(seed=11, vocab_size=512, concentration=2.0, logit_range=4.0)
    prompts = [[1 + r, 2 + r % 7, 3] for r in range(48)]
    res = {}
    for mode in ("1", "0"):
        monkeypatch.setenv("LCB_ENGINE_GRAPH", mode)
        eng = WaveEngine(model, 1 << 28, max_tokens=24, device=DEV)
        eng.register_agent("a")
        got = []
        for w in range(4):
            reqs = [GenerateRequest("a", p, lcb.SamplingConfig(temperature=0.8, top_p=0.9, max_tokens=24,
                                                               seed=1000 * w + r),
                                    lcb.ReplayPolicy.STEP_WISE if w % 2 == 0 else lcb.ReplayPolicy.NONE,
                                    request_id=f"{w}-{r}")
                    for r, p in enumerate(prompts)]
            got.append([(g.tokens, g.outcome.replayed_len, g.outcome.diverged_at, g.flags)
                        for g in eng.generate_wave(reqs)])
        ents = {d: (e.token_seq, np.asarray(e.logits_seq, np.float32).tobytes()) for d, e in eng.cache.entries.items()}
        res[mode] = (got, ents, len(eng._graphs))
    assert res["1"][0] == res["0"][0]
    assert res["1"][1] == res["0"][1]
    assert 1 <= res["1"][2] <= 4 and res["0"][2] == 0
