"""The reference's own hot-path unit tests, run against this package (drop-in proof).

Every case below restates one test of the reference suite for the path --
``pkg/tests/test_logits_cache.py`` (20-141) and ``pkg/tests/test_sampling.py``
(27-283) -- with the same inputs and the same assertions, but importing
``paper_2604_17353_b200`` where the reference imports ``agentserve``.  The
cache runs on the HBM slab / GPU index, the sampling functions on the CUDA
probability kernels (``lc_softmax``, ``lc_truncate_probs``, ``lc_draw_probs``,
``lc_row_entropy``).  Each test names the reference test it restates.

The reference's hypothesis properties run with fewer examples (each example is a
few kernel launches).
"""

from __future__ import annotations

import math

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

import paper_2604_17353_b200 as lcb
from paper_2604_17353_b200 import (
    TOKEN_OVERHEAD_BYTES,
    ConfigError,
    HotspotParams,
    LogitsCache,
    ReplayOutcome,
    RngStream,
    SamplingConfig,
    StateKey,
)

pytestmark = pytest.mark.gpu

S = lcb.sampling


def _traj(n, vocab=8, fill=0.0):
    """A constant (n, vocab) float32 trajectory and tokens 0..n-1 (test_logits_cache.py:16-17)."""
    return np.full((n, vocab), fill, dtype=np.float32), list(range(n))


def _entry_bytes(n, vocab):
    return n * vocab * 4 + n * TOKEN_OVERHEAD_BYTES


# ------------------------------------------------------------------ test_logits_cache.py


def test_cache_miss_on_empty():  # test_lookup_empty_cache (:20-22)
    assert LogitsCache().lookup(StateKey.of([1, 2, 3])) is None


def test_cache_roundtrip():  # test_write_then_read (:25-34)
    cache = LogitsCache()
    key = StateKey.of([1, 2])
    rows, toks = _traj(5)
    cache.update(key, rows, toks)
    hit = cache.lookup(key)
    assert hit is not None and len(hit) == 5
    assert hit.logits_seq.shape == (5, 8)
    assert hit.token_seq == toks


def test_cache_rejects_length_mismatch():  # test_update_rejects_mismatched_lengths (:37-41)
    rows, _ = _traj(5)
    with pytest.raises(ConfigError):
        LogitsCache().update(StateKey.of([1]), rows, [1, 2, 3])


def test_cache_accounting_500x256():  # test_size_accounting_500_tokens_vocab_256 (:44-49)
    cache = LogitsCache()
    e = cache.update(StateKey.of([1]), np.zeros((500, 256), dtype=np.float32), list(range(500)))
    assert e.nbytes == _entry_bytes(500, 256)
    assert cache.total_bytes == e.nbytes


def test_cache_overwrite_single_entry():  # test_overwrite_keeps_single_entry (:52-58)
    cache = LogitsCache()
    key = StateKey.of([7])
    cache.update(key, *_traj(4))
    cache.update(key, *_traj(6))
    assert len(cache) == 1 and len(cache.lookup(key)) == 6


@pytest.mark.parametrize("refresh_first", [True, False])
def test_cache_lru_eviction(refresh_first):
    """test_lru_eviction_over_budget (:61-72) with the refresh; test_capacity_eviction_after_fill
    (:75-81) without it: budget = two 4-row entries, the least recently hit goes first."""
    cache = LogitsCache(budget_bytes=2 * _entry_bytes(4, 8))
    keys = [StateKey.of([i]) for i in (1, 2, 3)]
    cache.update(keys[0], *_traj(4))
    cache.update(keys[1], *_traj(4))
    if refresh_first:
        cache.lookup(keys[0])
        cache.update(keys[2], *_traj(4))
        assert cache.lookup(keys[1]) is None
        assert cache.lookup(keys[0]) is not None and cache.lookup(keys[2]) is not None
    else:
        cache.update(keys[2], *_traj(4))
        assert cache.lookup(keys[0]) is None


def test_cache_pin_survives():  # test_pinned_entry_survives_eviction (:84-95)
    cache = LogitsCache(budget_bytes=2 * _entry_bytes(4, 8))
    keys = [StateKey.of([i]) for i in (1, 2, 3)]
    cache.update(keys[0], *_traj(4))
    held = cache.lookup(keys[0])
    cache.pin(held)
    cache.update(keys[1], *_traj(4))
    cache.update(keys[2], *_traj(4))
    assert cache.lookup(keys[0]) is not None
    cache.unpin(held)


def test_cache_hotspot_memo():  # test_hotspots_computed_once (:98-115)
    cache = LogitsCache()
    key = StateKey.of([5])
    rows = np.array([[4.0, 0.0, 0.0, 0.0], [1.0, 1.0, 0.8, 0.2], [5.0, 0.0, 0.0, 0.0]], dtype=np.float32)
    cache.update(key, rows, [0, 1, 0])
    e = cache.lookup(key)
    cfg, hp = SamplingConfig(temperature=1.0, max_tokens=1), HotspotParams()
    first = cache.hotspots_for(e, cfg, hp)
    assert cache.hotspot_computations == 1
    assert cache.hotspots_for(e, cfg, hp) == first and cache.hotspot_computations == 1
    cache.hotspots_for(e, cfg, HotspotParams(threshold=0.1))
    assert cache.hotspot_computations == 2


def test_cache_prefetch_missing_key():  # test_prefetch_on_missing_key_is_noop (:118-121)
    cache = LogitsCache()
    cache.prefetch(StateKey.of([9]), SamplingConfig(max_tokens=1), HotspotParams())
    assert cache.hotspot_computations == 0


def test_cache_prefetch_queue():  # test_prefetch_queue_drains (:124-136)
    cache = LogitsCache()
    key = StateKey.of([1])
    cfg, hp = SamplingConfig(temperature=1.0, max_tokens=1), HotspotParams()
    cache.update(key, *_traj(3), prefetch_config=(cfg, hp))
    assert cache.hotspot_computations == 0
    assert cache.drain_prefetch() == 1 and cache.hotspot_computations == 1
    assert cache.hotspots_for(cache.lookup(key), cfg, hp) is not None
    assert cache.hotspot_computations == 1


def test_replay_outcome_ratio():  # test_replay_outcome_hit_ratio (:139-141)
    assert ReplayOutcome(replayed_len=50, diverged_at=49, total_len=500, forward_passes_saved=50).hit_ratio == 0.1
    assert ReplayOutcome(0, None, 0, 0).hit_ratio == 0.0


# ------------------------------------------------------------------ test_sampling.py: softmax


def test_softmax_cases():
    """test_softmax_symmetric_pair (:30-32), _temperature_zero_is_greedy (:35-40),
    _matches_direct_exponentiation (:43-49), _temperature_scales_sharpness (:52-56)."""
    f32 = lambda *v: np.array(v, dtype=np.float32)  # noqa: E731
    assert np.allclose(S.softmax(f32(0.0, 0.0), 1.0), [0.5, 0.5], atol=0)
    assert S.softmax(f32(1.0, 0.0), 0.0).tolist() == [1.0, 0.0]
    assert S.softmax(f32(2.0, 2.0, 1.0), 0.0).tolist() == [1.0, 0.0, 0.0]
    p = S.softmax(f32(2.0, 1.0, 0.0), 1.0)
    den = math.exp(2.0) + math.exp(1.0) + 1.0
    assert np.allclose(p, [math.exp(2.0) / den, math.exp(1.0) / den, 1.0 / den], atol=1e-12)
    assert abs(p.sum() - 1.0) < 1e-9
    assert S.softmax(f32(1.0, 0.0), 0.25)[0] > S.softmax(f32(1.0, 0.0), 4.0)[0]


# ------------------------------------------------------------------ truncate


@pytest.mark.parametrize("p,k,top_p,want,exact", [
    ((0.5, 0.3, 0.2), 1, 1.0, [1.0, 0.0, 0.0], True),          # _top_k_single_survivor (:66-68)
    ((0.5, 0.3, 0.2), None, 0.7, [0.625, 0.375, 0.0], False),  # _top_p_hand_renormalized (:71-73)
    ((0.5, 0.5), None, 0.5, [1.0, 0.0], True),                 # _top_p_exact_boundary_kept (:76-78)
    ((0.25, 0.25, 0.25, 0.25), 2, 1.0, [0.5, 0.5, 0.0, 0.0], True),  # _tie_prefers_lower_token_id (:81-83)
    ((0.4, 0.3, 0.2, 0.1), 3, 0.5, [4 / 7, 3 / 7, 0.0, 0.0], False),  # _composes_top_k_then_top_p (:86-89)
])
def test_truncate_known_answers(p, k, top_p, want, exact):
    out = S.truncate(np.array(p, dtype=np.float64), k, top_p)
    if exact:
        assert out.tolist() == want
    else:
        assert np.allclose(out, want, atol=1e-12)


def test_truncate_unconstrained_is_identity():  # test_truncate_identity_when_unconstrained (:60-63)
    p = np.array([0.5, 0.3, 0.2])
    assert np.array_equal(S.truncate(p, None, 1.0), p)


@given(st.lists(st.floats(min_value=0.01, max_value=1.0), min_size=2, max_size=16),
       st.floats(min_value=0.05, max_value=1.0))
@settings(max_examples=40, deadline=None)
def test_truncate_distribution_property(weights, top_p):  # test_truncate_keeps_valid_distribution (:92-103)
    p = np.array(weights) / sum(weights)
    out = S.truncate(p, None, top_p)
    assert abs(out.sum() - 1.0) < 1e-9 and np.all(out >= 0)
    assert np.count_nonzero(out) <= np.count_nonzero(p)


# ------------------------------------------------------------------ sample


def test_sample_one_hot_one_value():  # test_sample_one_hot_consumes_one_value (:126-130)
    rs = RngStream(1)
    assert S.sample(np.array([0.0, 1.0, 0.0]), rs) == 1 and rs.position == 1


def test_sample_frequencies_two_way():
    """test_sample_two_way_frequencies (:133-141): 100k draws of RngStream(31337) on [0.5, 0.5],
    as one batched launch (same uniforms in the same order as 100k sequential calls)."""
    n = 100_000
    rs = RngStream(31337)
    u = np.array([rs.next_float() for _ in range(n)])
    import torch

    d = lcb._dev.device()
    p = torch.tensor([[0.5, 0.5]], dtype=torch.float64, device=d).expand(n, 2).contiguous()
    ut = torch.from_numpy(u).to(d)
    tok = torch.empty(n, dtype=torch.int32, device=d)
    fl = torch.empty(n, dtype=torch.uint8, device=d)
    lcb._capi.check(lcb._capi.lib.lc_draw_probs(p.data_ptr(), 2, n, 2, ut.data_ptr(), tok.data_ptr(), fl.data_ptr(),
                                                lcb._dev.stream_ptr(d)), "lc_draw_probs")
    counts = np.bincount(tok.cpu().numpy(), minlength=2)
    assert abs(counts[0] / n - 0.5) < 0.01 and abs(counts[1] / n - 0.5) < 0.01
    # the first few equal the sequential single-call path
    rs2 = RngStream(31337)
    assert [S.sample(np.array([0.5, 0.5]), rs2) for _ in range(16)] == tok[:16].cpu().tolist()


def test_sample_seed_determinism():  # test_sample_deterministic_given_seed (:144-150)
    p = np.array([0.2, 0.3, 0.5])
    a, b = RngStream(42), RngStream(42)
    assert [S.sample(p, a) for _ in range(50)] == [S.sample(p, b) for _ in range(50)]


def test_sample_zero_mass_raises():  # test_sample_rejects_zero_mass (:153-155)
    with pytest.raises(RuntimeError):
        S.sample(np.array([0.0, 0.0]), RngStream(1))


def test_sample_skips_zero_probability():  # test_sample_never_returns_zero_prob_token (:158-162)
    rs = RngStream(5)
    p = np.array([0.7, 0.0, 0.3])
    assert all(S.sample(p, rs) != 1 for _ in range(300))


# ------------------------------------------------------------------ entropy / max_prob / hotspots


def test_entropy_and_max_prob_cases():
    """test_entropy_uniform_and_one_hot (:168-170), _hand_case (:173-176), test_max_prob_cases (:179-182)."""
    assert abs(S.entropy(np.full(4, 0.25)) - math.log(4)) < 1e-12
    assert S.entropy(np.array([0.0, 1.0, 0.0])) == 0.0
    want = -(0.75 * math.log(0.75) + 0.25 * math.log(0.25))
    assert abs(S.entropy(np.array([0.75, 0.25])) - want) < 1e-12 and abs(want - 0.5623) < 1e-4
    assert S.max_prob(np.array([0.0, 1.0])) == 1.0
    assert S.max_prob(np.full(4, 0.25)) == 0.25
    assert S.max_prob(np.array([0.6, 0.3, 0.1])) == 0.6


@given(st.lists(st.floats(min_value=0.001, max_value=1.0), min_size=2, max_size=64))
@settings(max_examples=40, deadline=None)
def test_entropy_range_property(weights):  # test_entropy_bounds (:185-190)
    p = np.array(weights) / sum(weights)
    assert -1e-12 <= S.entropy(p) <= math.log(len(p)) + 1e-12


def test_hotspot_score_cases():
    """test_hotspot_score_zero_for_one_hot (:196-199), _decay_ratio (:202-207),
    _uniform_hand_value (:210-213), _rejects_negative_step (:216-218)."""
    hp = HotspotParams()
    assert S.hotspot_score(np.array([0.0, 1.0]), 0, hp) == 0.0
    assert S.hotspot_score(np.array([1.0, 0.0]), 123, hp) == 0.0
    p = np.array([0.5, 0.25, 0.25])
    r = S.hotspot_score(p, 0, HotspotParams(decay=0.1)) / S.hotspot_score(p, 10, HotspotParams(decay=0.1))
    assert abs(r - 2.0) < 1e-12
    assert abs(S.hotspot_score(np.full(4, 0.25), 0, HotspotParams(decay=0.37)) - math.log(4) * 0.75) < 1e-12
    with pytest.raises(ConfigError):
        S.hotspot_score(np.array([0.5, 0.5]), -1, hp)


def test_hotspots_of_one_hot_rows_empty():  # test_identify_hotspots_all_one_hot_is_empty (:230-233)
    rows = []
    for i in range(6):
        z = np.full(4, -30.0, dtype=np.float32)
        z[i % 4] = 30.0
        rows.append(z)
    assert S.identify_hotspots(rows, SamplingConfig(temperature=1.0, max_tokens=1), HotspotParams()) == ()


def test_select_hotspots_threshold_cap():  # test_select_hotspots_threshold_and_cap (:236-242)
    sc = np.array([0.9, 0.3, 0.7])
    assert S.select_hotspots(sc, HotspotParams(threshold=0.6)) == (0, 2)
    assert S.select_hotspots(sc, HotspotParams(threshold=0.6, max_hotspots=1)) == (0,)


def test_identify_hotspots_vs_plain_math():  # test_identify_hotspots_matches_direct_oracle (:245-272)
    rs = RngStream(2718)
    rows = [np.array([rs.next_float() * 6 - 3 for _ in range(8)], dtype=np.float32) for _ in range(40)]
    T, decay, thr = 0.8, 0.015, 0.55
    raw = []
    for t, z in enumerate(rows):
        s = [float(v) / T for v in z]
        mx = max(s)
        ex = [math.exp(v - mx) for v in s]
        tot = sum(ex)
        p = [v / tot for v in ex]
        h = -sum(v * math.log(v) for v in p if v > 0)
        raw.append(h * (1 - max(p)) / (1 + decay * t))
    lo, hi = min(raw), max(raw)
    want = tuple(t for t in range(len(raw)) if (raw[t] - lo) / (hi - lo) > thr)
    got = S.identify_hotspots(rows, SamplingConfig(temperature=T, max_tokens=1), HotspotParams(decay=decay, threshold=thr))
    assert got == want


@given(st.floats(min_value=0.01, max_value=100.0))
@settings(max_examples=25, deadline=None)
def test_select_hotspots_scale_property(scale):  # test_select_hotspots_rescale_invariant (:275-283)
    hp = HotspotParams(threshold=0.6)
    sc = np.array([0.02, 0.9, 0.33, 0.7, 0.0, 0.55])
    assert S.select_hotspots(sc * scale, hp) == S.select_hotspots(sc, hp)
