"""Pin the CPU oracle against golden vectors produced by the reference itself.

Mirrors the reference's own hot-path unit tests (pkg/tests/test_mixing.py,
test_kernels.py, test_sampling.py, test_logits_cache.py) but checks the
oracle restatement in ``oracle/`` instead, so the GPU parity tests can trust
it as the checker.
"""

from __future__ import annotations

import math

import numpy as np
import pytest

from oracle import cache_ref, mixing_ref, sampling_ref
from tests.golden_io import load_json, sampling_cases


# -- mixing (test_mixing.py:16-49, determinism.md:36-39) -------------------------------


def test_avalanche_frozen_values():
    assert mixing_ref.avalanche64(0) == 0
    assert mixing_ref.avalanche64(1) == 0x5692161D100B05E5
    assert mixing_ref.avalanche64(0x9E3779B97F4A7C15) == 0xE220A8397B1DCDAF


def test_mixing_golden():
    g = load_json("mixing.json")
    for v, a in g["avalanche"]:
        assert mixing_ref.avalanche64(v) == a
        assert int(mixing_ref.avalanche64_np(np.array([v], dtype=np.uint64))[0]) == a
    for a, b, m in g["mix2"]:
        assert mixing_ref.mix2(a, b) == m
    for seq, h in g["hash"]:
        assert mixing_ref.hash_tokens(seq) == h
    for seed, us in g["uniform"]:
        assert [mixing_ref.uniform(seed, i) for i in range(len(us))] == us
        got = mixing_ref.uniforms_np([seed] * len(us), np.arange(len(us)))
        assert got.tolist() == us


def test_anchor_values_from_survey():
    # SURVEY.md 8(c) anchors measured on the reference
    assert mixing_ref.hash_tokens([1, 2, 3]) == 0xA8765FB996CEE2D4
    assert [mixing_ref.uniform(0, i) for i in range(3)] == [0.6362254214077777, 0.5895323551334491, 0.7452038393704972]


def test_prefix_extension_property():
    toks = [3, 1, 4, 1, 5, 9, 2, 6]
    assert mixing_ref.hash_tokens(toks + [7]) == mixing_ref.fold_token(mixing_ref.hash_tokens(toks), 7)
    assert mixing_ref.hash_tokens(toks[4:], mixing_ref.hash_tokens(toks[:4])) == mixing_ref.hash_tokens(toks)


def test_fill_logits_golden():
    g = load_json("mixing.json")
    for vocab, state, conc, rng, want in g["fill"]:
        row = mixing_ref.fill_logits_np(state, vocab, conc, rng)
        bits = row.view(np.uint32)
        if vocab <= 1000:
            assert bits.tolist() == want
        else:
            assert int(bits.sum(dtype=np.uint64)) == want[0]
            assert bits[:4].tolist() == want[1]


# -- sampling (test_sampling.py) --------------------------------------------------------


def test_sampling_golden_tokens_and_kept_sets():
    n = 0
    for c in sampling_cases():
        q = sampling_ref.truncate(sampling_ref.softmax(c.z, c.T), c.top_k, c.top_p)
        assert np.array_equal(np.flatnonzero(q > 0), c.kept), c.name
        for u, tok in zip(c.u, c.tokens):
            assert sampling_ref.draw(q, float(u)) == tok, (c.name, u)
            n += 1
        if c.q is not None:
            assert np.array_equal(q, c.q), c.name
    assert n > 4000


def test_probs_golden_cases():
    g = load_json("probs.json")
    for case in g["cases"]:
        p = np.array(case["p"])
        q = sampling_ref.truncate(p, case["top_k"], case["top_p"])
        assert q.tolist() == case["q"]
        for u, tok in case["draws"]:
            assert sampling_ref.draw(q, u) == tok
    assert g["zero_mass"] == "RuntimeError"
    with pytest.raises(RuntimeError):
        sampling_ref.draw(np.zeros(2), 0.5)


def test_truncate_hand_cases():
    P = lambda *v: np.array(v, dtype=np.float64)  # noqa: E731
    assert sampling_ref.truncate(P(0.5, 0.3, 0.2), 1, 1.0).tolist() == [1.0, 0.0, 0.0]
    assert np.allclose(sampling_ref.truncate(P(0.5, 0.3, 0.2), None, 0.7), [0.625, 0.375, 0.0], atol=1e-12)
    assert sampling_ref.truncate(P(0.5, 0.5), None, 0.5).tolist() == [1.0, 0.0]
    assert sampling_ref.truncate(P(0.25, 0.25, 0.25, 0.25), 2, 1.0).tolist() == [0.5, 0.5, 0.0, 0.0]
    assert np.allclose(sampling_ref.truncate(P(0.4, 0.3, 0.2, 0.1), 3, 0.5), [4 / 7, 3 / 7, 0, 0], atol=1e-12)
    # full-distribution mass rule (SURVEY.md hard part 2)
    assert np.count_nonzero(sampling_ref.truncate(P(0.5, 0.3, 0.2), 2, 0.55)) == 2
    assert sampling_ref.draw(P(0.2, 0, 0.8, 0), 0.2) == 2
    assert sampling_ref.draw(P(0.2, 0, 0.8, 0), 0.0) == 0


def test_survey_model_anchor():
    z = mixing_ref.fill_logits_np(mixing_ref.mix2(7, mixing_ref.hash_tokens([1, 2, 3])), 32000, 2.5, 5.0)
    assert int(np.argmax(z)) == 29475
    assert float(z.max()) == 12.287679672241211
    assert abs(sampling_ref.softmax(z, 0.6).max() - 0.989961) < 1e-6


def test_hotspots_golden():
    for case in load_json("hotspots.json"):
        rows = np.array(case["rows"], dtype=np.uint32).view(np.float32)
        hs = sampling_ref.identify_hotspots(list(rows), case["T"], case["decay"], case["threshold"], case["max_hotspots"])
        assert list(hs) == case["hotspots"]


def test_entropy_hand_case():
    expected = -(0.75 * math.log(0.75) + 0.25 * math.log(0.25))
    assert abs(sampling_ref.entropy(np.array([0.75, 0.25])) - expected) < 1e-12


# -- cache (test_logits_cache.py + reference traces) -------------------------------------


def test_cache_oracle_replays_reference_traces():
    for tr in load_json("cache_traces.json"):
        cache = cache_ref.CacheOracle(tr["budget"], key_capacity=64, page_capacity=4096)
        handles = {}
        for op in tr["ops"]:
            kind, digest = op[0], op[1]
            state = op[-1]
            if kind == "lookup":
                e = cache.lookup(digest)
                assert (e is not None) == op[2]
            elif kind == "update":
                e, _ = cache.insert(digest, op[2], op[3])
                handles[digest] = (e.slot, e.gen)
            elif kind == "pin":
                e = cache.entries[digest]
                cache.pin(e.slot, e.gen)
            elif kind == "unpin":
                e = cache.entries[digest]
                cache.unpin(e.slot, e.gen)
            assert sorted(cache.entries) == state["present"]
            assert cache.total == state["total"]
            assert cache.hits == state["hits"] and cache.lookups == state["lookups"]


def test_cache_oracle_lru_and_pins():
    one = 4 * 8 * 4 + 4 * 8
    c = cache_ref.CacheOracle(2 * one, 16, 64)
    c.insert(1, 4, 8)
    c.insert(2, 4, 8)
    c.lookup(1)
    _, victims = c.insert(3, 4, 8)
    assert [v[0] for v in victims] == [2]
    # slot discipline: LIFO reuse of the evicted slot
    e4, _ = c.insert(4, 4, 8)
    assert e4.slot == 1  # slot of key 2 was freed before key 4 needed one


def test_cache_oracle_heap_mode_equals_scan_mode():
    """The O(log E) victim heap used at C4 scale picks the reference's victims."""
    rng = np.random.default_rng(3)
    one = 2 * 16 * 4 + 2 * 8
    a = cache_ref.CacheOracle(12 * one, 64, 512, 2)
    b = cache_ref.CacheOracle(12 * one, 64, 512, 2, heap=True)
    for step in range(3000):
        d = int(rng.integers(0, 40))
        r = rng.random()
        if r < 0.3:
            ea, eb = a.lookup(d), b.lookup(d)
            assert (ea is None) == (eb is None)
            if ea is not None:
                assert ea.slot == eb.slot
        elif r < 0.4 and a.entries:
            e = a.entries[sorted(a.entries)[int(rng.integers(0, len(a.entries)))]]
            delta = 1 if (e.pins == 0 or rng.random() < 0.5) else -1
            a.pin(e.slot, e.gen, delta)
            b.pin(e.slot, e.gen, delta)
        else:
            n = int(rng.integers(1, 4))
            ea, va = a.insert(d, n, 16)
            eb, vb = b.insert(d, n, 16)
            assert (ea.slot, ea.gen, ea.pages) == (eb.slot, eb.gen, eb.pages)
            assert va == vb
        assert a.total == b.total and sorted(a.entries) == sorted(b.entries)


def test_fast_kept_order_and_draw_many_equal_the_reference_order():
    """oracle.sampling_ref.kept_order_fast / draw_many (bulk-check helpers) == the
    reference-order kept_order / per-draw draw on producer rows and golden cases."""
    rng = np.random.default_rng(0)
    cases = [(mixing_ref.fill_logits_np(mixing_ref.mix2(5, i), V, conc, 5.0), T, k, p)
             for i, (V, conc, T, k, p) in enumerate([(32000, 2.5, 0.6, None, 0.9), (32000, 0.0, 0.6, None, 0.9),
                                                      (32000, 0.0, 1.0, None, 0.99), (20000, 2.5, 0.6, 50, 0.95),
                                                      (20000, 0.0, 1.0, 50, 0.95), (9000, 1.0, 0.3, 7000, 1.0),
                                                      (9000, 0.0, 2.0, None, 0.999), (512, 0.0, 1.0, 40, 0.2)])]
    for c in sampling_cases()[::7]:
        cases.append((c.z, c.T, c.top_k, c.top_p))
    for z, T, k, p in cases:
        prob = sampling_ref.softmax(z, T)
        a, b = sampling_ref.kept_order(prob, k, p), sampling_ref.kept_order_fast(prob, k, p, cand=256)
        assert (a is None and b is None) or np.array_equal(a, b), (T, k, p)
        q = sampling_ref.truncate(prob, k, p)
        q2, K = sampling_ref.truncate_fast(prob, k, p)
        assert np.array_equal(q, q2) and K == (len(z) if a is None else len(a))
        us = np.concatenate([rng.random(40), [0.0, 1.0 - 2 ** -53]])
        assert sampling_ref.draw_many(q, us).tolist() == [sampling_ref.draw(q, float(u)) for u in us]


def test_bulk_check_counts_and_catches_mismatches():
    from oracle import bulk

    V, n, D = 2048, 6, 5
    states = np.array([mixing_ref.mix2(7, i) for i in range(n)], dtype=np.uint64)
    seeds = np.array([[mixing_ref.mix2(1, 10 * r + b) for b in range(D)] for r in range(n)], dtype=np.uint64)
    index = np.arange(n)
    toks, kept = [], []
    for r in range(n):
        z = mixing_ref.bf16_round(mixing_ref.fill_logits_np(int(states[r]), V, 2.5, 5.0))
        prob = sampling_ref.softmax(z, 0.6)
        q = sampling_ref.truncate(prob, None, 0.9)
        toks.append([sampling_ref.draw(q, mixing_ref.uniform(int(seeds[r, b]), r)) for b in range(D)])
        kept.append(len(sampling_ref.kept_order(prob, None, 0.9)))
    toks, kept = np.array(toks, np.int32), np.array(kept, np.int32)
    job = dict(V=V, T=0.6, k=None, p=0.9, bf16=True, conc=2.5, states=states, seeds=seeds, index=index,
               tokens=toks, kept=kept)
    r = bulk.check_rows(job)
    assert (r["draws"], r["token_mismatches"], r["kept_checked"], r["kept_mismatches"]) == (n * D, 0, n, 0)
    toks[2, 3] += 1
    kept[4] += 1
    r = bulk.check_rows(dict(job, tokens=toks, kept=kept))
    assert r["token_mismatches"] == 1 and r["kept_mismatches"] == 1
