"""Cache-interface edge cases (round-2 review findings), on the GPU:

* entries narrower than the slab are replayed over their own width;
* replay buffers are rebuilt when a caller reuses them for another shape;
* a rebuild (wider / longer entry) keeps pins and rounds and makes old handles stale;
* generation-checked reads: a handle whose entry was overwritten reads nothing;
* slab-page exhaustion rolls the insert back exactly like the oracle (no leaked slot).
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import cache_ref, mixing_ref, sampling_ref

pytestmark = pytest.mark.gpu

lcb = pytest.importorskip("paper_2604_17353_b200")

DEV = torch.device("cuda", 0)


def _oracle_tok(z, T, k, p, u):
    return sampling_ref.draw(sampling_ref.truncate(sampling_ref.softmax(z, T), k, p), float(u))


def _params(n, T=0.6, k=0, p=0.9):
    return (torch.full((n,), T, dtype=torch.float64, device=DEV), torch.full((n,), k, dtype=torch.int32, device=DEV),
            torch.full((n,), p, dtype=torch.float64, device=DEV))


@pytest.mark.parametrize("dtype", ["float32", "bfloat16"])
def test_replay_of_entries_narrower_than_the_slab(dtype):
    Vs, Vn, n_req, L, nb = 4096, 1000, 5, 12, 3
    cache = lcb.LogitsCache(1 << 30, vocab=Vs, dtype=dtype, max_rows=16)
    keys = [mixing_ref.hash_tokens([r, 1, 2]) for r in range(n_req)]
    rows = mixing_ref.fill_rows_np([mixing_ref.mix2(8, i) for i in range(n_req * L)], Vn, 2.5)
    if dtype == "bfloat16":
        rows = mixing_ref.bf16_round(rows)
    # first write a wide entry under every key so the slab pages hold large stale values, then
    # overwrite with the narrow entries (an unfixed replay would sample the stale columns)
    wide = np.full((n_req * L, Vs), 50.0, np.float32)
    tdt = torch.bfloat16 if dtype == "bfloat16" else torch.float32
    dig = lcb._dev.u64_tensor(keys, DEV)
    lens = torch.full((n_req,), L, dtype=torch.int32, device=DEV)
    offs = torch.arange(n_req, dtype=torch.int64, device=DEV) * L
    cache.insert_batch(dig, lens, torch.full((n_req,), Vs, dtype=torch.int32, device=DEV),
                       torch.from_numpy(wide).to(DEV).to(tdt), offs, torch.zeros(n_req * L, dtype=torch.int32,
                                                                                 device=DEV), L)
    toks = rows.argmax(1).astype(np.int32)
    cache.insert_batch(dig, lens, torch.full((n_req,), Vn, dtype=torch.int32, device=DEV),
                       torch.from_numpy(rows).to(DEV).to(tdt), offs, torch.from_numpy(toks).to(DEV), L)
    seeds = [mixing_ref.mix2(3, b) for b in range(n_req * nb)]
    kept = torch.zeros(n_req * L, dtype=torch.int32, device=DEV)
    tok, rep, div, slot, ln = cache.replay_stepwise(dig, L, nb, lcb._dev.u64_tensor(seeds, DEV), *_params(n_req),
                                                    kept=kept)
    tok = tok.cpu().numpy().reshape(n_req, L, nb)
    rep = rep.cpu().numpy().reshape(n_req, nb)
    kept = kept.cpu().numpy()
    for r in range(n_req):
        for b in range(nb):
            for t in range(int(rep[r, b])):
                u = mixing_ref.uniform(seeds[r * nb + b], t)
                assert tok[r, t, b] == _oracle_tok(rows[r * L + t], 0.6, None, 0.9, u), (r, b, t)
        assert np.all(kept[r * L:(r + 1) * L] <= Vn)


def test_replay_buffers_rebuilt_on_shape_change():
    V, n_req, L = 2048, 4, 10
    cache = lcb.LogitsCache(1 << 30, vocab=V, dtype="bfloat16", max_rows=16)
    keys = [mixing_ref.hash_tokens([r, 7]) for r in range(n_req)]
    rows = mixing_ref.bf16_round(mixing_ref.fill_rows_np([mixing_ref.mix2(4, i) for i in range(n_req * L)], V, 2.5))
    cache.insert_batch(lcb._dev.u64_tensor(keys, DEV), torch.full((n_req,), L, dtype=torch.int32, device=DEV),
                       torch.full((n_req,), V, dtype=torch.int32, device=DEV),
                       torch.from_numpy(rows).to(DEV).to(torch.bfloat16),
                       torch.arange(n_req, dtype=torch.int64, device=DEV) * L,
                       torch.from_numpy(rows.argmax(1).astype(np.int32)).to(DEV), L)
    dig = lcb._dev.u64_tensor(keys, DEV)
    bufs = {}
    for max_pos, nb in ((8, 2), (4, 5), (10, 5), (3, 1)):
        seeds = lcb._dev.u64_tensor([mixing_ref.mix2(5, b) for b in range(n_req * nb)], DEV)
        a = [x.clone() for x in cache.replay_stepwise(dig, max_pos, nb, seeds, *_params(n_req), bufs=bufs)[:3]]
        f = cache.replay_stepwise(dig, max_pos, nb, seeds, *_params(n_req))[:3]
        for x, y in zip(a, f):
            assert torch.equal(x, y), (max_pos, nb)


def test_rebuild_keeps_pins_and_makes_old_handles_stale():
    cache = lcb.LogitsCache(1 << 30, max_rows=4)
    ka, kb = lcb.StateKey.of([1, 2]), lcb.StateKey.of([3])
    za = np.arange(3 * 32, dtype=np.float32).reshape(3, 32)
    cache.update(ka, za, [5, 6, 7], round_index=4)
    ea = cache.lookup(ka)
    cache.pin(ea)
    assert ea.pins == 1
    cache.update(kb, np.ones((6, 64), np.float32), list(range(6)))  # wider AND longer: rebuild
    with pytest.raises(lcb.ConfigError):
        ea.logits_seq  # noqa: B018 -- the pre-rebuild handle is stale
    ea2 = cache.lookup(ka)
    assert ea2.pins == 1 and ea2.created_round == 4
    assert np.array_equal(ea2.logits_seq, za) and ea2.token_seq == [5, 6, 7]
    assert len(cache) == 2 and cache.lookups == 2 and cache.hits == 2
    cache.unpin(ea2)
    assert ea2.pins == 0


def test_overwritten_handle_reads_nothing():
    cache = lcb.LogitsCache(1 << 30, vocab=16, max_rows=4)
    k = lcb.StateKey.of([9])
    cache.update(k, np.ones((2, 16), np.float32), [1, 2])
    old = cache.lookup(k)
    cache.update(k, np.full((2, 16), 3.0, np.float32), [3, 4])
    assert old.token_seq == [-1, -1]
    assert not old.logits_seq.any()
    new = cache.lookup(k)
    assert new.token_seq == [3, 4] and np.all(new.logits_seq == 3.0)


@pytest.mark.parametrize("scalar", [False, True])
def test_page_exhaustion_rolls_back_like_the_oracle(scalar, monkeypatch):
    """A budget that admits more (narrow) rows than the slab holds: inserts that find no pages are
    rolled back (key out of the index, slot reusable) -- slots, live map and accounting equal the
    oracle's, and the latched error surfaces as CapacityError."""
    if scalar:
        monkeypatch.setenv("LCB_SCALAR_POLICY", "1")
    V, E, P, pr = 64, 64, 10, 2
    cache = lcb.LogitsCache(1 << 40, vocab=V, key_capacity=E, page_rows=pr, max_rows=8, page_capacity=P)
    orc = cache_ref.CacheOracle(1 << 40, E, P, pr)
    rng = np.random.default_rng(2)
    errors = 0
    for step in range(12):
        keys = rng.integers(1, 30, 3).tolist()
        lens = rng.integers(1, 7, 3).astype(np.int32)
        want = []
        for d, n in zip(keys, lens):
            e, _ = orc.insert(int(d), int(n), V)
            want.append(-1 if e is None else e.slot)
        rows = torch.zeros((int(lens.sum()), V), dtype=torch.float32, device=DEV)
        offs = np.concatenate([[0], np.cumsum(lens)[:-1]]).astype(np.int64)
        slot, _ = cache.insert_batch(lcb._dev.u64_tensor(keys, DEV), torch.from_numpy(lens).to(DEV),
                                     torch.full((3,), V, dtype=torch.int32, device=DEV), rows,
                                     torch.from_numpy(offs).to(DEV),
                                     torch.zeros(int(lens.sum()), dtype=torch.int32, device=DEV), 6)
        assert slot.cpu().tolist() == want, step
        try:
            st = cache._stats()
        except lcb.CapacityError:
            errors += 1
            st = cache._stats()
        assert (st.entries, st.total_bytes, st.free_pages) == (len(orc.entries), orc.total, len(orc.free_pages))
        snap = cache._snapshot()
        live = {int(snap["digest"][s]): int(s) for s in np.flatnonzero(snap["alive"])}
        assert live == {d: e.slot for d, e in orc.entries.items()}, step
    assert errors > 0 and orc.capacity_errors > 0
