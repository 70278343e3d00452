"""Hotspot scoring kept beside the cached rows and selection on the device
against the oracle's restatement of the reference (sampling.py:112-160, numpy fp64) at the
C1 scale: V = 32000, 500-row trajectories, decay 0.001, threshold 0.6 (tot_default.json)."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import mixing_ref, sampling_ref

pytestmark = pytest.mark.gpu

lcb = pytest.importorskip("paper_2604_17353_b200")

DEV = torch.device("cuda", 0)


def _cache_with(rows_per_entry, V, dtype, max_rows):
    n_ent = len(rows_per_entry)
    cache = lcb.LogitsCache(1 << 36, vocab=V, dtype=dtype, max_rows=max_rows, key_capacity=n_ent + 64)
    keys = [mixing_ref.mix2(31, i) for i in range(n_ent)]
    lens = [len(r) for r in rows_per_entry]
    flat = np.concatenate(rows_per_entry)
    offs = np.concatenate([[0], np.cumsum(lens)[:-1]]).astype(np.int64)
    t = torch.from_numpy(flat).to(DEV)
    if dtype == "bfloat16":
        t = t.to(torch.bfloat16)
    cache.insert_batch(lcb._dev.u64_tensor(keys, DEV), torch.tensor(lens, dtype=torch.int32, device=DEV),
                       torch.full((n_ent,), V, dtype=torch.int32, device=DEV), t, torch.from_numpy(offs).to(DEV), None,
                       max(lens))
    return cache, keys


@pytest.mark.parametrize("dtype,max_hot", [("float32", None), ("float32", 5), ("bfloat16", None)])
def test_hotspots_match_oracle_at_c1_scale(dtype, max_hot):
    V, n_ent, L = 32000, 10, 500
    T, decay, thr = 0.6, 0.001, 0.6
    ents = []
    for e in range(n_ent):
        rows = mixing_ref.fill_rows_np([mixing_ref.mix2(7, e * L + t) for t in range(L)], V, 2.5)
        if dtype == "bfloat16":
            rows = mixing_ref.bf16_round(rows)
        ents.append(rows)
    cache, keys = _cache_with(ents, V, dtype, L)
    cfg = lcb.SamplingConfig(temperature=T, max_tokens=L)
    hp = lcb.HotspotParams(decay=decay, threshold=thr, max_hotspots=max_hot)
    n_total = 0
    for k, rows in zip(keys, ents):
        e = cache.lookup(lcb.StateKey(k))
        got = cache.hotspots_for(e, cfg, hp)
        want = sampling_ref.identify_hotspots(rows, T, decay, thr, max_hot)
        assert list(got) == list(want)
        n_total += len(want)
    assert n_total > 0 and cache.hotspot_uncertain == 0
    # the batched device path (replay layout) agrees with the per-entry tuples
    slot, gen, ln, vv = cache.lookup_batch(lcb._dev.u64_tensor(keys, DEV))
    di, nh, fl = cache.hotspot_draw_index_device(slot, gen, L, T, hp)
    di = di.view(n_ent, L).cpu().numpy()
    for i, rows in enumerate(ents):
        want = sampling_ref.identify_hotspots(rows, T, decay, thr, max_hot)
        assert list(np.flatnonzero(di[i] >= 0)) == list(want)
        assert list(di[i][di[i] >= 0]) == list(range(len(want)))
        assert int(nh[i]) == len(want)
    assert int(fl.max()) == 0


def test_hotspot_edge_entries():
    """Exactly one-hot rows (every score exactly 0): span 0, no hotspots, nothing uncertain;
    a dead handle is flagged; T = 0 scores are exactly 0."""
    V, L = 64, 12
    rows = np.full((L, V), -1e4, dtype=np.float32)  # every other exp(s) underflows to 0: exactly one-hot
    rows[np.arange(L), np.arange(L) % V] = 1e4
    cache, keys = _cache_with([rows], V, "float32", L)
    e = cache.lookup(lcb.StateKey(keys[0]))
    cfg = lcb.SamplingConfig(temperature=1.0, max_tokens=L)
    assert cache.hotspots_for(e, cfg, lcb.HotspotParams()) == ()
    assert cache.hotspots_for(e, lcb.SamplingConfig(temperature=0.0, max_tokens=L), lcb.HotspotParams()) == ()
    assert cache.hotspot_uncertain == 0
    slot = torch.tensor([e.slot], dtype=torch.int32, device=DEV)
    gen = torch.tensor([e.gen + 1], dtype=torch.int64, device=DEV).to(torch.int32)  # a stale handle
    di, nh, fl = cache.hotspot_draw_index_device(slot, gen, L, 1.0, lcb.HotspotParams())
    assert int(fl[0]) & 4 and int(nh[0]) == 0 and bool((di < 0).all())


def test_scores_survive_writeback_prefix_and_go_stale_on_rewrite():
    """A row keeps its score until it is rewritten: re-selection after an unrelated insert
    needs no rescoring (same tuple), an overwrite with new rows rescoring gives the new
    rows' hotspots."""
    V, L = 256, 40
    a = mixing_ref.fill_rows_np([mixing_ref.mix2(3, t) for t in range(L)], V, 1.0)
    b = mixing_ref.fill_rows_np([mixing_ref.mix2(4, t) for t in range(L)], V, 1.0)
    cache, keys = _cache_with([a], V, "float32", L)
    cfg = lcb.SamplingConfig(temperature=0.8, max_tokens=L)
    hp = lcb.HotspotParams(decay=0.01, threshold=0.5)
    e = cache.lookup(lcb.StateKey(keys[0]))
    assert list(cache.hotspots_for(e, cfg, hp)) == list(sampling_ref.identify_hotspots(a, 0.8, 0.01, 0.5))
    e2 = cache.update(lcb.StateKey(keys[0]), b, list(range(L)))
    slot = torch.tensor([e2.slot], dtype=torch.int32, device=DEV)
    gen = torch.tensor([e2.gen], dtype=torch.int64, device=DEV).to(torch.int32)
    di, nh, fl = cache.hotspot_draw_index_device(slot, gen, L, 0.8, hp, score=False)
    assert int(fl[0]) & 2  # the rewritten rows are not scored yet
    di, nh, fl = cache.hotspot_draw_index_device(slot, gen, L, 0.8, hp)
    assert int(fl[0]) == 0
    assert list(np.flatnonzero(di.cpu().numpy() >= 0)) == list(sampling_ref.identify_hotspots(b, 0.8, 0.01, 0.5))
