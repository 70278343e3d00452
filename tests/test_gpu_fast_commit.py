"""The batched fast commit of the insert policy (lc_cache.cu commit_kernel: parallel
start-of-batch records + one committing thread + the hash-edit log warp) vs the oracle
allocator, and vs the warp policy it hands over to (LCB_FAST_COMMIT=0): slots, generations,
victims, hit/miss, accounting, the live map and the slab rows of every live entry.

The cases drive every hand-over: duplicates in a batch (overwrite of an entry made earlier in
the same batch), overwrites of start-of-batch entries, entries of 0 rows and of narrower vocab
(several evictions per insert), batches that evict every start-of-batch entry and then their
own inserts (candidates used up -> the warp resumes inside an insert's eviction loop), pinned
entries met at the LRU end (side list -> the warp policy takes the next batches) and page
exhaustion (the warp latches the error and rolls back).
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import cache_ref, mixing_ref

pytestmark = pytest.mark.gpu

lcb = pytest.importorskip("paper_2604_17353_b200")
from paper_2604_17353_b200 import _capi  # noqa: E402

DEV = torch.device("cuda", 0)


def _pin(cache, orc, slot, gen, delta):
    orc.pin(slot, gen, delta)
    st_ = torch.tensor([slot], dtype=torch.int32, device=DEV)
    gt_ = torch.tensor([gen], dtype=torch.int64, device=DEV).to(torch.int32)
    _capi.check(_capi.lib.lc_cache_pin(cache.handle, st_.data_ptr(), gt_.data_ptr(), 1, delta, cache._stream()))
    cache._dirty()


@pytest.mark.parametrize("mode", ["fast", "warp"])
@pytest.mark.parametrize("page_rows,max_rows,narrow,pins", [(1, 1, False, False), (4, 4, True, False),
                                                            (1, 1, True, True), (2, 2, False, True)])
def test_fast_commit_vs_oracle(mode, page_rows, max_rows, narrow, pins, monkeypatch):
    if mode == "warp":
        monkeypatch.setenv("LCB_FAST_COMMIT", "0")
    rng = np.random.default_rng(100 + 7 * page_rows + 3 * narrow + pins)
    V, E = 32, 1024
    budget = (V * 4 + 8) * max_rows * 150
    cache = lcb.LogitsCache(budget, vocab=V, key_capacity=E, page_rows=page_rows, max_rows=max_rows,
                            page_capacity=E)
    assert cache.max_pages == 1
    orc = cache_ref.CacheOracle(budget, E, E, page_rows)
    keys = [mixing_ref.mix2(17, k) for k in range(700)]
    row_id = 0
    expect = {}
    pinned = []
    for step in range(70):
        r = rng.random()
        if r < 0.2:
            batch = [keys[int(i)] for i in rng.integers(0, len(keys), int(rng.integers(1, 200)))]
            slot = cache.lookup_batch(lcb._dev.u64_tensor(batch, DEV))[0]
            assert slot.cpu().tolist() == [-1 if (e := orc.lookup(d)) is None else e.slot for d in batch], step
        if pins and rng.random() < 0.15 and orc.entries:
            if pinned and rng.random() < 0.4:
                sl, g = pinned.pop(int(rng.integers(0, len(pinned))))
                _pin(cache, orc, sl, g, -1)
            elif len(pinned) < 8:
                e = orc.entries[list(orc.entries)[int(rng.integers(0, len(orc.entries)))]]
                pinned.append((e.slot, e.gen))
                _pin(cache, orc, e.slot, e.gen, 1)
        # mostly batches within the budget; now and then one larger than the whole cache
        nb = int(rng.integers(1, 260)) if rng.random() < 0.85 else int(rng.integers(300, 600))
        batch = [keys[int(i)] for i in rng.integers(0, len(keys), nb)]
        lens = rng.integers(0, max_rows + 1, nb).astype(np.int32)
        vocs = (rng.integers(1, V + 1, nb) if narrow else np.full(nb, V)).astype(np.int32)
        offs = np.concatenate([[0], np.cumsum(lens)[:-1]]).astype(np.int64)
        tot = max(int(lens.sum()), 1)
        ids = row_id + np.arange(tot)
        rows = (ids[:, None] * 64 + np.arange(V)[None, :]).astype(np.float32)
        slot, gen = cache.insert_batch(lcb._dev.u64_tensor(batch, DEV), torch.from_numpy(lens).to(DEV),
                                       torch.from_numpy(vocs).to(DEV), torch.from_numpy(rows).to(DEV),
                                       torch.from_numpy(offs).to(DEV), torch.from_numpy(ids.astype(np.int32)).to(DEV),
                                       max_rows)
        want_s, want_g = [], []
        for d, n, v, o in zip(batch, lens, vocs, offs):
            e, _ = orc.insert(d, int(n), int(v))
            want_s.append(e.slot)
            want_g.append(e.gen)
            expect[d] = (row_id + int(o), int(v))
        assert slot.cpu().tolist() == want_s, step
        assert (gen.cpu().numpy().astype(np.int64) & 0xFFFFFFFF).tolist() == want_g, step
        row_id += tot
        st = cache._stats()
        assert (st.entries, st.total_bytes, st.hits, st.lookups, st.evictions) == (
            len(orc.entries), orc.total, orc.hits, orc.lookups, orc.evictions), step
        snap = cache._snapshot()
        live = {int(snap["digest"][s]): int(s) for s in np.flatnonzero(snap["alive"])}
        assert live == {d: e.slot for d, e in orc.entries.items()}, step
        if step % 10 == 9:
            for d, e in orc.entries.items():
                if e.n == 0:
                    continue
                r0, v = expect[d]
                got = cache._gather(e.slot, e.gen, e.n, v).cpu().numpy()
                rr = r0 + np.arange(e.n)
                assert np.array_equal(got[:, :v], (rr[:, None] * 64 + np.arange(v)[None, :]).astype(np.float32)), d
    assert orc.evictions > 2000


def test_fast_commit_equals_warp_policy_on_a_long_trace(monkeypatch):
    """The C4 shape at small scale (single-row entries, 90% inserts of uniform keys, a full
    cache): the fast commit and the warp policy give the same slots for every op of the trace."""
    V, E, K = 16, 20000, 60000
    budget = (V * 4 + 8) * (E - 64)
    rng = np.random.default_rng(3)
    keys = torch.tensor(np.array([mixing_ref.mix2(5, k) for k in range(K)], dtype=np.uint64).view(np.int64),
                        device=DEV)
    ops = [(rng.integers(0, K, 400), rng.integers(0, K, 3600)) for _ in range(40)]
    outs = {}
    for mode in ("fast", "warp"):
        if mode == "warp":
            monkeypatch.setenv("LCB_FAST_COMMIT", "0")
        cache = lcb.LogitsCache(budget, vocab=V, key_capacity=E, page_rows=1, max_rows=1, page_capacity=E)
        got = []
        for lk, ins in ops:
            got.append(cache.lookup_batch(keys[torch.from_numpy(lk).to(DEV)])[0].cpu().numpy())
            n = len(ins)
            s, g = cache.insert_batch(keys[torch.from_numpy(ins).to(DEV)], torch.ones(n, dtype=torch.int32, device=DEV),
                                      torch.full((n,), V, dtype=torch.int32, device=DEV),
                                      torch.zeros((1, V), device=DEV), torch.zeros(n, dtype=torch.int64, device=DEV),
                                      None, 1)
            got.append(s.cpu().numpy())
            got.append(g.cpu().numpy())
        st = cache._stats()
        outs[mode] = (np.concatenate(got), (st.entries, st.total_bytes, st.hits, st.evictions))
    assert np.array_equal(outs["fast"][0], outs["warp"][0])
    assert outs["fast"][1] == outs["warp"][1]
    assert outs["fast"][1][3] > 50000
