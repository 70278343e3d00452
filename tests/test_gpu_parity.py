"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle and the
reference's golden vectors.  Bit-exact for tokens, kept sets, hashes,
uniforms, hit/miss and slots; probabilities within 1e-5 relative (fp32) --
the tolerance BASELINE.json's north star states.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import cache_ref, mixing_ref, sampling_ref
from tests.golden_io import load_json, sampling_cases

pytestmark = pytest.mark.gpu

lcb = pytest.importorskip("paper_2604_17353_b200")
from paper_2604_17353_b200 import _capi  # noqa: E402

DEV = torch.device("cuda", 0)


def _resample_rows(rows: np.ndarray, T, k, p, u_lists, dtype=torch.float32):
    """One task per row; row i draws u_lists[i]."""
    z = torch.from_numpy(np.ascontiguousarray(rows, dtype=np.float32)).to(DEV).to(dtype)
    n = len(rows)
    counts = np.array([len(x) for x in u_lists])
    begin = np.concatenate([[0], np.cumsum(counts)[:-1]])
    tasks = lcb.make_tasks(row=np.arange(n), temperature=T, top_k=k, top_p=p, draw_begin=begin,
                           draw_end=begin + counts)
    u = torch.tensor(np.concatenate(u_lists), dtype=torch.float64, device=DEV)
    cnt = torch.zeros(8, dtype=torch.int64, device=DEV)
    tok, fl = lcb.resample(z, tasks, u=u, counters=cnt)
    return tok.cpu().numpy(), fl.cpu().numpy(), cnt.cpu().numpy()


# -- mixing ----------------------------------------------------------------------------


def test_hash_prefix_golden():
    g = load_json("mixing.json")
    seqs = [s for s, _ in g["hash"]]
    got = lcb.mixing.hash_prompts(seqs)
    assert [int(x) for x in got.cpu().numpy().view(np.uint64)] == [h for _, h in g["hash"]]
    # prefix extension from a parent digest
    toks = list(range(1, 300))
    par = lcb.mixing.hash_prompts([toks[:100]])
    ext = lcb.mixing.hash_prompts([toks[100:]], parents=par.cpu().numpy().view(np.uint64))
    assert int(ext.cpu().numpy().view(np.uint64)[0]) == mixing_ref.hash_tokens(toks)


def test_uniforms_golden():
    g = load_json("mixing.json")
    for seed, us in g["uniform"]:
        got = lcb.uniforms([seed] * len(us), np.arange(len(us))).cpu().numpy()
        assert got.tolist() == us


def test_fill_logits_matches_reference_producer():
    g = load_json("mixing.json")
    for vocab, state, conc, rng, want in g["fill"]:
        st = lcb._dev.u64_tensor([state], DEV)
        out = torch.empty(vocab, dtype=torch.float32, device=DEV)
        _capi.check(_capi.lib.lc_fill_logits(st.data_ptr(), 1, vocab, conc, rng, _capi.LC_F32, out.data_ptr(), vocab,
                                             None))
        bits = out.cpu().numpy().view(np.uint32)
        if vocab <= 1000:
            assert bits.tolist() == want
        else:
            assert int(bits.sum(dtype=np.uint64)) == want[0] and bits[:4].tolist() == want[1]
        outb = torch.empty(vocab, dtype=torch.bfloat16, device=DEV)
        _capi.check(_capi.lib.lc_fill_logits(st.data_ptr(), 1, vocab, conc, rng, _capi.LC_BF16, outb.data_ptr(),
                                             vocab, None))
        ref = mixing_ref.bf16_round(mixing_ref.fill_logits_np(state, vocab, conc, rng))
        assert np.array_equal(outb.float().cpu().numpy(), ref)



@pytest.mark.parametrize("vocab,conc,rng", [(32000, 2.5, 5.0), (151936, 2.5, 5.0), (1003, 1.7, -3.25),
                                            (4099, 0.5, 1e-3), (77, 2.5, 1e-300)])
def test_fill_logits_many_rows_match_oracle(vocab, conc, rng):
    """The vectorised producer (8 ids per thread, one DFMA per value, packed bf16 rounding) against
    the oracle's numpy restatement of the reference fill, bit for bit, over many rows: peaks in every
    position of an 8-id group, ragged tails (V % 8), a negative and a tiny range (scalar path)."""
    n = 24
    states = [mixing_ref.mix2(91, i) for i in range(n)]
    st = lcb._dev.u64_tensor(states, DEV)
    for dt, tdt in ((_capi.LC_F32, torch.float32), (_capi.LC_BF16, torch.bfloat16)):
        out = torch.empty((n, vocab), dtype=tdt, device=DEV)
        _capi.check(_capi.lib.lc_fill_logits(st.data_ptr(), n, vocab, conc, rng, dt, out.data_ptr(), vocab, None))
        got = out.float().cpu().numpy()
        for i, s_ in enumerate(states):
            want = mixing_ref.fill_logits_np(s_, vocab, conc, rng)
            if dt == _capi.LC_BF16:
                want = mixing_ref.bf16_round(want)
            assert np.array_equal(got[i].view(np.uint32), want.view(np.uint32)), (vocab, dt, i)


# -- fast-tier error model ------------------------------------------------------------------


def _probe(z, m, T, mode):
    zt = torch.from_numpy(z).to(DEV)
    out = torch.empty(z.size, dtype=torch.float64, device=DEV)
    _capi.check(_capi.lib.lc_probe_exp(zt.data_ptr(), z.size, float(m), T, mode, out.data_ptr(), None))
    return out.cpu().numpy()


@pytest.mark.parametrize("mode,bound", [(0, 4.0e-7), (2, 3.0e-13)])
def test_exp_error_bounds(mode, bound):
    """The constants kEx2RelErr (mode 0) and kLiteErr (mode 2) in lc_resample.cu
    must bound the tiers' exponentials (relative to exp((z-m)/T) in fp64)."""
    rng = np.random.default_rng(mode)
    worst = 0.0
    for T in (0.01, 0.1, 0.6, 1.0, 1.3, 7.0):
        m = np.float32(rng.normal() * 4)
        z = (m - rng.random(1 << 20) * 60 * T).astype(np.float32)
        z[:1024] = np.nextafter(m, np.float32(-np.inf), dtype=np.float32) - np.arange(1024, dtype=np.float32) * 1e-6
        got = _probe(z, m, T, mode)
        # exact argument in extended precision: (z - m) exact in f64, then / T
        exact = np.exp((z.astype(np.longdouble) - np.longdouble(m)) / np.longdouble(T)).astype(np.float64)
        ok = exact > 1e-37
        worst = max(worst, float((np.abs(got[ok] - exact[ok]) / exact[ok]).max()))
    assert worst < bound, worst


def test_cheap_exp_error_model():
    """cheap_exp: |e - exact| <= exact * (kEx2Raw + kArgRel*|a|) (+ flushed subnormals)."""
    rng = np.random.default_rng(7)
    kEx2Raw, kArgRel = 2.5e-7, 3.0 * 2.0 ** -24 * np.log(2) * 1.01
    for T in (0.05, 0.6, 1.0, 3.0):
        m = np.float32(rng.normal() * 4)
        z = (m - rng.random(1 << 20) * 80 * T).astype(np.float32)
        got = _probe(z, m, T, 1)
        a = (z.astype(np.longdouble) - np.longdouble(m)) / np.longdouble(T) / np.log(np.longdouble(2))
        exact = np.exp2(a).astype(np.float64)
        ok = exact > 2e-38
        bound = exact[ok] * (kEx2Raw + kArgRel * np.abs(a[ok].astype(np.float64)))
        assert np.all(np.abs(got[ok] - exact[ok]) <= bound)


def test_ex2_raw_bound():
    """ex2.approx alone (a = 0 offset, exact arguments): max relative error < kEx2Raw."""
    x = np.linspace(-125.0, 0.0, 1 << 22).astype(np.float32)
    got = _probe(x, np.float32(0.0), 1.0 / np.log(2.0), 1)  # L = 1 exactly -> a = x
    exact = np.exp2(x.astype(np.float64))
    assert float((np.abs(got - exact) / exact).max()) < 2.5e-7


def test_bf16_ex2_bound():
    """ex2.approx.ftz.bf16x2 over every non-positive bf16 input down to -126:
    relative error (incl. the bf16 rounding of the result) well inside
    kEx2Bf16Err = 0.01 (lc_stage.cu FAST exit bound)."""
    h = np.arange(0x8000, 0x10000, dtype=np.uint32)  # negative bf16 bit patterns
    x = (h << 16).view(np.float32)
    x = x[np.isfinite(x) & (x >= -126.0)]
    x = np.concatenate([x, np.float32([0.0])])
    got = _probe(x, np.float32(0.0), 1.0, 3)
    exact = np.exp2(x.astype(np.float64))
    worst = float((np.abs(got - exact) / exact).max())
    assert worst < 0.008, worst


# -- resample vs golden (reference) ----------------------------------------------------------


@pytest.mark.parametrize("as_bf16", [False, True])
def test_resample_golden_cases(as_bf16):
    cases = sampling_cases()
    if as_bf16:  # rows that are exactly bf16-representable can go through the bf16 kernels
        cases = [c for c in cases if c.name.startswith("bf16_")]
    n_checked = 0
    for c in cases:
        tok, fl, _ = _resample_rows(c.z[None, :], c.T, c.top_k, c.top_p, [c.u],
                                    dtype=torch.bfloat16 if as_bf16 else torch.float32)
        assert tok.tolist() == c.tokens.tolist(), (c.name, c.T, c.top_k, c.top_p)
        assert not np.any(fl & _capi.LC_DRAW_UNRESOLVED), (c.name, c.T, c.top_k, c.top_p, c.u, fl)
        n_checked += len(c.u)
    assert n_checked > (500 if as_bf16 else 4000)


@pytest.mark.parametrize("tier", ["precise", "exact"])
def test_forced_tiers_match_golden(tier, monkeypatch):
    """Every task through the PRECISE pass / the EXACT kernel (LCB_FORCE_TIER hook)."""
    monkeypatch.setenv("LCB_FORCE_TIER", tier)
    cases = [c for c in sampling_cases() if len(c.z) <= 4099]
    for c in cases:
        tok, fl, _ = _resample_rows(c.z[None, :], c.T, c.top_k, c.top_p, [c.u])
        assert tok.tolist() == c.tokens.tolist(), (tier, c.name, c.T, c.top_k, c.top_p)
    rows = mixing_ref.bf16_round(mixing_ref.fill_rows_np([mixing_ref.mix2(17, i) for i in range(6)], 32000, 0.0))
    ul = [np.random.default_rng(i).random(4).tolist() for i in range(6)]
    for T, k, p in ((0.6, None, 0.9), (1.0, 50, 0.95), (0.6, None, 1.0)):
        tok, _, _ = _resample_rows(rows, T, k, p, ul, dtype=torch.bfloat16)
        assert tok.tolist() == _oracle_tokens(rows, T, k, p, ul), (tier, T, k, p)


def _oracle_tokens(rows, T, k, p, ulists):
    out = []
    for z, us in zip(rows, ulists):
        q = sampling_ref.truncate(sampling_ref.softmax(z, T), k, p)
        out += [sampling_ref.draw(q, float(u)) for u in us]
    return out


@pytest.mark.parametrize("V,conc,T,k,p,bf16", [
    (32000, 2.5, 0.6, None, 1.0, False),   # config 1 shape (fp32, untruncated)
    (32000, 2.5, 0.6, None, 0.9, True),    # config 2 shape (bf16, top-p 0.9)
    (32000, 0.0, 0.6, None, 0.9, True),    # flat worst case: large nucleus
    (32000, 0.0, 1.0, None, 1.0, False),
    (151936, 2.5, 0.6, 50, 0.95, True),    # configs 3/5 shape
    (128256, 2.5, 0.6, None, 1.0, True),
    (4099, 1.0, 0.25, 3, 0.999, False),
])
def test_resample_matches_oracle(V, conc, T, k, p, bf16):
    rng = np.random.default_rng(V + int(conc * 10) + int(T * 100))
    nrows = 24 if V > 100000 else 64
    states = [mixing_ref.mix2(7, 10_000 + i) for i in range(nrows)]
    rows = mixing_ref.fill_rows_np(states, V, conc)
    if bf16:
        rows = mixing_ref.bf16_round(rows)
    ulists = [rng.random(8).tolist() + [0.0] for _ in range(nrows)]
    tok, fl, cnt = _resample_rows(rows, T, k, p, ulists, dtype=torch.bfloat16 if bf16 else torch.float32)
    want = _oracle_tokens(rows, T, k, p, ulists)
    assert tok.tolist() == want
    assert not np.any(fl & _capi.LC_DRAW_UNRESOLVED)


def test_resample_large_nucleus_many_draws():
    """Flat rows (large nucleus) with 32 draws each: exercises the bracket / kept-list
    path and its PRECISE / EXACT fallbacks."""
    V = 32000
    rng = np.random.default_rng(99)
    rows = mixing_ref.bf16_round(mixing_ref.fill_rows_np([mixing_ref.mix2(13, i) for i in range(24)], V, 0.0))
    ulists = [rng.random(32).tolist() for _ in range(24)]
    for T, p in ((0.6, 0.9), (1.0, 0.95), (0.3, 0.5)):
        tok, fl, cnt = _resample_rows(rows, T, None, p, ulists, dtype=torch.bfloat16)
        assert tok.tolist() == _oracle_tokens(rows, T, None, p, ulists), (T, p, cnt)


def test_seed_mode_uniforms_equal_explicit_u():
    V = 1000
    rows = mixing_ref.fill_rows_np([mixing_ref.mix2(3, i) for i in range(16)], V, 1.0)
    seeds = [mixing_ref.mix2(1, b) for b in range(4)]
    # task t (row t, position pos=t) draws 4 branches with u = uniform(seed_b, t)
    tasks = lcb.make_tasks(row=np.arange(16), pos=np.arange(16), temperature=0.8, top_p=0.9,
                           draw_begin=np.arange(16) * 4, draw_end=np.arange(16) * 4 + 4, seed_base=0)
    z = torch.from_numpy(rows).to(DEV)
    sd = lcb._dev.u64_tensor(seeds, DEV)
    tok, _ = lcb.resample(z, tasks, seeds=sd, n_draws=64)
    want = []
    for t in range(16):
        for b in range(4):
            want += _oracle_tokens(rows[t:t + 1], 0.8, None, 0.9, [[mixing_ref.uniform(seeds[b], t)]])
    assert tok.cpu().tolist() == want


def test_edge_rows():
    # NaN row is flagged; -inf entries are zero-probability; T == 0 is greedy
    z = np.array([[1.0, np.nan, 0.0, 2.0], [-np.inf, 3.0, -np.inf, 3.0], [5.0, 5.0, 1.0, -1.0]], dtype=np.float32)
    tok, fl, _ = _resample_rows(z, 1.0, None, 1.0, [[0.5], [0.1, 0.9], [0.3]])
    assert tok[0] == -1 and fl[0] & _capi.LC_DRAW_BAD_ROW
    want = _oracle_tokens(z[1:], 1.0, None, 1.0, [[0.1, 0.9], [0.3]])
    assert tok[1:].tolist() == want
    tok0, _, _ = _resample_rows(z[2:], 0.0, 2, 0.5, [[0.0, 0.99]])
    assert tok0.tolist() == [0, 0]


def test_many_draws_per_row_shared():
    """Best-of-N sharing: 64 draws per row in one task == oracle."""
    V = 32000
    rows = mixing_ref.bf16_round(mixing_ref.fill_rows_np([mixing_ref.mix2(9, i) for i in range(8)], V, 2.5))
    rng = np.random.default_rng(5)
    ulists = [rng.random(64).tolist() for _ in range(8)]
    tok, _, _ = _resample_rows(rows, 0.6, None, 0.9, ulists, dtype=torch.bfloat16)
    assert tok.tolist() == _oracle_tokens(rows, 0.6, None, 0.9, ulists)


# -- probability-level API -------------------------------------------------------------------


def test_probs_api_golden():
    g = load_json("probs.json")
    for case in g["cases"]:
        p = np.array(case["p"])
        q = lcb.truncate(p, case["top_k"], case["top_p"])
        assert np.asarray(q).tolist() == case["q"]
        for u, tok in case["draws"]:
            class U:
                def next_float(self, u=u):
                    return u
            assert lcb.sample(np.asarray(q), U()) == tok
    with pytest.raises(RuntimeError):
        lcb.sample(np.zeros(2), lcb.RngStream(1))


def test_softmax_matches_oracle():
    for V, T in ((3, 1.0), (64, 0.6), (32000, 0.6), (1000, 0.0)):
        z = mixing_ref.fill_logits_np(mixing_ref.mix2(2, V), V, 2.5, 5.0)
        got = lcb.softmax(z, T)
        want = sampling_ref.softmax(z, T)
        assert np.allclose(got, want, rtol=1e-12, atol=0)


def test_hotspots_golden():
    for case in load_json("hotspots.json"):
        rows = np.array(case["rows"], dtype=np.uint32).view(np.float32)
        cfg = lcb.SamplingConfig(temperature=case["T"], max_tokens=1)
        hp = lcb.HotspotParams(decay=case["decay"], threshold=case["threshold"], max_hotspots=case["max_hotspots"])
        assert list(lcb.identify_hotspots(list(rows), cfg, hp)) == case["hotspots"]


@pytest.mark.parametrize("dtype", ["float32", "bfloat16"])
def test_cache_hotspots_from_slab_match_golden(dtype):
    """hotspots_for scores the entry's rows in place (lc_cache_row_entropy) -- same hotspots as
    the reference's identify_hotspots on the same rows (golden cases), and the same scores as
    row_scores on the gathered rows."""
    for case in load_json("hotspots.json"):
        rows = np.array(case["rows"], dtype=np.uint32).view(np.float32)
        if dtype == "bfloat16":
            rows = mixing_ref.bf16_round(rows)
        n, V = rows.shape
        cache = lcb.LogitsCache(1 << 30, vocab=V, dtype=dtype, max_rows=max(n, 1))
        cache.insert_batch(lcb._dev.u64_tensor([77], DEV), torch.tensor([n], dtype=torch.int32, device=DEV),
                           torch.tensor([V], dtype=torch.int32, device=DEV), torch.from_numpy(rows).to(DEV),
                           torch.zeros(1, dtype=torch.int64, device=DEV), None, n)
        e = cache.lookup(lcb.StateKey(77))
        cfg = lcb.SamplingConfig(temperature=case["T"], max_tokens=1)
        hp = lcb.HotspotParams(decay=case["decay"], threshold=case["threshold"], max_hotspots=case["max_hotspots"])
        got = cache.row_scores(e, case["T"], case["decay"])
        want = lcb.sampling.row_scores(e.logits_device(), case["T"], case["decay"], DEV)
        assert np.array_equal(got, want)
        assert list(cache.hotspots_for(e, cfg, hp)) == list(lcb.identify_hotspots(list(rows), cfg, hp))
        if dtype == "float32":
            assert list(cache.hotspots_for(e, cfg, hp)) == case["hotspots"]


# -- cache ---------------------------------------------------------------------------------------


def test_cache_replays_reference_traces():
    for tr in load_json("cache_traces.json"):
        cache = lcb.LogitsCache(tr["budget"], vocab=16, key_capacity=64, max_rows=8)
        pinned = {}
        for op in tr["ops"]:
            kind, digest, state = op[0], op[1], op[-1]
            if kind == "lookup":
                e = cache.lookup(lcb.StateKey(digest))
                assert (e is not None) == op[2]
            elif kind == "update":
                n, v = op[2], op[3]
                cache.update(lcb.StateKey(digest), np.zeros((n, v), np.float32), list(range(n)))
            elif kind == "pin":
                e = cache.entries[digest]
                cache.pin(e)
            elif kind == "unpin":
                e = cache.entries[digest]
                cache.unpin(e)
            assert sorted(cache.entries) == state["present"], kind
            assert cache.total_bytes == state["total"]
            assert cache.hits == state["hits"] and cache.lookups == state["lookups"]


def test_cache_slots_match_oracle_under_batches():
    """Batched inserts/lookups: hit/miss, slots and victims bit-exact vs the oracle allocator."""
    rng = np.random.default_rng(42)
    V, page_rows = 64, 4
    one = 6 * V * 4 + 6 * 8
    budget = one * 20
    cache = lcb.LogitsCache(budget, vocab=V, key_capacity=128, page_rows=page_rows, max_rows=8, page_capacity=256)
    orc = cache_ref.CacheOracle(budget, 128, 256, page_rows)
    keys = [mixing_ref.hash_tokens([i, 77]) for i in range(60)]
    for step in range(40):
        nb = int(rng.integers(1, 24))
        batch = [keys[int(i)] for i in rng.integers(0, len(keys), nb)]
        if rng.random() < 0.5:
            dg = lcb._dev.u64_tensor(batch, DEV)
            slot, gen, ln, vv = cache.lookup_batch(dg)
            want = []
            for d in batch:
                e = orc.lookup(d)
                want.append(-1 if e is None else e.slot)
            assert slot.cpu().tolist() == want
        else:
            lens = rng.integers(0, 8, nb).astype(np.int32)
            offs = np.concatenate([[0], np.cumsum(lens)[:-1]]).astype(np.int64)
            tot = int(lens.sum()) or 1
            rows = torch.randn(tot, V, device=DEV)
            toks = torch.arange(tot, dtype=torch.int32, device=DEV)
            slot, gen = cache.insert_batch(lcb._dev.u64_tensor(batch, DEV), torch.from_numpy(lens).to(DEV),
                                           torch.full((nb,), V, dtype=torch.int32, device=DEV), rows,
                                           torch.from_numpy(offs).to(DEV), toks, int(lens.max()))
            want = [orc.insert(d, int(n), V)[0].slot for d, n in zip(batch, lens)]
            assert slot.cpu().tolist() == want
        st = cache._stats()
        assert st.entries == len(orc.entries)
        assert st.total_bytes == orc.total
        assert st.hits == orc.hits and st.lookups == orc.lookups
        snap = cache._snapshot()
        live = {int(snap["digest"][s]): int(s) for s in np.flatnonzero(snap["alive"])}
        assert live == {d: e.slot for d, e in orc.entries.items()}


@pytest.mark.parametrize("collide,page_rows,max_rows", [(False, 1, 1), (True, 4, 8), (False, 1, 40), (True, 1, 3),
                                                         (False, 16, 64)])
def test_cache_warp_policy_stress_vs_oracle(collide, page_rows, max_rows):
    """The warp policy kernel (register control block, windowed probes, ring windows, stack
    mirrors, scalar fallbacks) vs the oracle allocator: slots, generations, victims, hit/miss,
    accounting and the slab rows of every live entry, under duplicates in a batch, pins
    (side list), probe chains longer than the 32-bucket window and entries over 32 pages."""
    rng = np.random.default_rng(11 + page_rows + max_rows)
    V, E = 32, 128
    maxp = -(-max_rows // page_rows)
    budget = (V * 4 + 8) * 3 * max_rows
    cache = lcb.LogitsCache(budget, vocab=V, key_capacity=E, page_rows=page_rows, max_rows=max_rows,
                            page_capacity=E * maxp)
    orc = cache_ref.CacheOracle(budget, E, E * maxp, page_rows)
    if collide:  # one home bucket for every key (home = d & mask for d < 2^29): chains of 60
        keys = [5 + 256 * k for k in range(1, 61)]
    else:
        keys = [mixing_ref.mix2(3, k) for k in range(60)]
    row_id = 0
    expect = {}  # digest -> first row id of its live entry
    pinned = []
    for step in range(120):
        r = rng.random()
        if r < 0.25:
            batch = [keys[int(i)] for i in rng.integers(0, len(keys), int(rng.integers(1, 12)))]
            slot, gen, ln, vv = cache.lookup_batch(lcb._dev.u64_tensor(batch, DEV))
            want = [-1 if (e := orc.lookup(d)) is None else e.slot for d in batch]
            assert slot.cpu().tolist() == want
        elif r < 0.35 and orc.entries:
            if pinned and rng.random() < 0.5:
                sl, g = pinned.pop(int(rng.integers(0, len(pinned))))
                delta = -1
            else:
                e = orc.entries[list(orc.entries)[int(rng.integers(0, len(orc.entries)))]]
                sl, g = e.slot, e.gen
                if len(pinned) >= 6:
                    continue
                pinned.append((sl, g))
                delta = 1
            orc.pin(sl, g, delta)
            st_ = torch.tensor([sl], dtype=torch.int32, device=DEV)
            gt_ = torch.tensor([g], dtype=torch.int64, device=DEV).to(torch.int32)
            _capi.check(_capi.lib.lc_cache_pin(cache.handle, st_.data_ptr(), gt_.data_ptr(), 1, delta,
                                               cache._stream()))
            cache._dirty()
        else:
            nb = int(rng.integers(1, 40))
            batch = [keys[int(i)] for i in rng.integers(0, len(keys), nb)]
            lens = rng.integers(1, max_rows + 1, nb).astype(np.int32)
            offs = np.concatenate([[0], np.cumsum(lens)[:-1]]).astype(np.int64)
            tot = int(lens.sum())
            ids = row_id + np.arange(tot)
            rows = (ids[:, None] * 64 + np.arange(V)[None, :]).astype(np.float32)
            slot, gen = cache.insert_batch(lcb._dev.u64_tensor(batch, DEV), torch.from_numpy(lens).to(DEV),
                                           torch.full((nb,), V, dtype=torch.int32, device=DEV),
                                           torch.from_numpy(rows).to(DEV), torch.from_numpy(offs).to(DEV),
                                           torch.from_numpy(ids.astype(np.int32)).to(DEV), max_rows)
            want_s, want_g = [], []
            for d, n, o in zip(batch, lens, offs):
                e, _ = orc.insert(d, int(n), V)
                want_s.append(e.slot)
                want_g.append(e.gen)
                expect[d] = row_id + int(o)
            assert slot.cpu().tolist() == want_s
            assert (gen.cpu().numpy().astype(np.int64) & 0xFFFFFFFF).tolist() == want_g
            row_id += tot
        st = cache._stats()
        assert (st.entries, st.total_bytes, st.hits, st.lookups) == (len(orc.entries), orc.total, orc.hits,
                                                                     orc.lookups), step
        assert st.evictions == orc.evictions
        snap = cache._snapshot()
        live = {int(snap["digest"][s]): int(s) for s in np.flatnonzero(snap["alive"])}
        assert live == {d: e.slot for d, e in orc.entries.items()}, step
        if step % 15 == 14:
            for d, e in orc.entries.items():
                got = cache._gather(e.slot, e.gen, e.n, V).cpu().numpy()
                ids = expect[d] + np.arange(e.n)
                assert np.array_equal(got, (ids[:, None] * 64 + np.arange(V)[None, :]).astype(np.float32)), d
    assert orc.evictions > 20


def test_cache_warp_policy_large_batches_vs_oracle():
    """Batches of hundreds of inserts (many 32-key chunks, duplicates within a batch, several
    evictions per batch spanning many LRU windows) interleaved with lookups and pins: slots and
    generations bit-exact vs the oracle, accounting and the live map equal after every batch."""
    rng = np.random.default_rng(5)
    V, E = 16, 4096
    budget = (V * 4 + 8) * 900
    cache = lcb.LogitsCache(budget, vocab=V, key_capacity=E, page_rows=1, max_rows=1, page_capacity=E)
    orc = cache_ref.CacheOracle(budget, E, E, 1)
    keys = [mixing_ref.mix2(9, k) for k in range(3000)]
    pinned = []
    for step in range(30):
        if rng.random() < 0.3:
            batch = [keys[int(i)] for i in rng.integers(0, len(keys), int(rng.integers(1, 400)))]
            slot = cache.lookup_batch(lcb._dev.u64_tensor(batch, DEV))[0]
            want = [-1 if (e := orc.lookup(d)) is None else e.slot for d in batch]
            assert slot.cpu().tolist() == want
        if rng.random() < 0.3 and orc.entries:
            ds = list(orc.entries)
            for _ in range(int(rng.integers(1, 6))):
                e = orc.entries[ds[int(rng.integers(0, len(ds)))]]
                delta = -1 if (e.slot, e.gen) in pinned and rng.random() < 0.5 else 1
                if delta == 1:
                    pinned.append((e.slot, e.gen))
                else:
                    pinned.remove((e.slot, e.gen))
                orc.pin(e.slot, e.gen, delta)
                st_ = torch.tensor([e.slot], dtype=torch.int32, device=DEV)
                gt_ = torch.tensor([e.gen], dtype=torch.int64, device=DEV).to(torch.int32)
                _capi.check(_capi.lib.lc_cache_pin(cache.handle, st_.data_ptr(), gt_.data_ptr(), 1, delta,
                                                   cache._stream()))
            cache._dirty()
        nb = int(rng.integers(100, 700))
        batch = [keys[int(i)] for i in rng.integers(0, len(keys), nb)]
        rows = torch.zeros((nb, V), dtype=torch.float32, device=DEV)
        slot, gen = cache.insert_batch(lcb._dev.u64_tensor(batch, DEV), torch.ones(nb, dtype=torch.int32, device=DEV),
                                       torch.full((nb,), V, dtype=torch.int32, device=DEV), rows,
                                       torch.arange(nb, dtype=torch.int64, device=DEV), None, 1)
        want = [orc.insert(d, 1, V)[0] for d in batch]
        assert slot.cpu().tolist() == [e.slot for e in want], step
        assert (gen.cpu().numpy().astype(np.int64) & 0xFFFFFFFF).tolist() == [e.gen for e in want], step
        st = cache._stats()
        assert (st.entries, st.total_bytes, st.hits, st.lookups, st.evictions) == (
            len(orc.entries), orc.total, orc.hits, orc.lookups, orc.evictions), step
        snap = cache._snapshot()
        live = {int(snap["digest"][s]): int(s) for s in np.flatnonzero(snap["alive"])}
        assert live == {d: e.slot for d, e in orc.entries.items()}, step
    assert orc.evictions > 3000


def test_miss_path_producer_resample_insert_then_replay():
    """The C3-sweep miss path end to end at a small size: producer rows (lc_fill_logits) ->
    resample with the branch seeds -> insert; the tokens equal the oracle's draws on the
    bf16 producer rows, and a later replay of the same keys hits, reads back the same rows
    and cached tokens, and (same seeds, draw number = position) replays every position."""
    V, n, R = 4096, 12, 6
    cache = lcb.LogitsCache(1 << 30, vocab=V, dtype="bfloat16", max_rows=R, page_rows=2)
    keys = [mixing_ref.hash_tokens([7, 7, j]) for j in range(n)]
    states = [mixing_ref.mix2(7, 1000 + i) for i in range(n * R)]
    rows = torch.empty((n * R, V), dtype=torch.bfloat16, device=DEV)
    st = lcb._dev.u64_tensor(states, DEV)
    _capi.check(_capi.lib.lc_fill_logits(st.data_ptr(), n * R, V, 2.5, 5.0, _capi.LC_BF16, rows.data_ptr(), V, None))
    ref_rows = mixing_ref.bf16_round(mixing_ref.fill_rows_np(states, V, 2.5))
    assert np.array_equal(rows.float().cpu().numpy(), ref_rows)
    seeds = [mixing_ref.mix2(1, j) for j in range(n)]
    tasks = lcb.make_tasks(row=np.arange(n * R), pos=np.tile(np.arange(R), n), temperature=0.6, top_k=50,
                           top_p=0.95, draw_begin=np.arange(n * R), draw_end=np.arange(n * R) + 1,
                           seed_base=np.repeat(np.arange(n), R))
    tok, _ = lcb.resample(rows, tasks, seeds=lcb._dev.u64_tensor(seeds, DEV), n_draws=n * R)
    tok = tok.cpu().numpy()
    for j in range(n):
        for t in range(R):
            u = mixing_ref.uniform(seeds[j], t)
            assert tok[j * R + t] == _oracle_tokens(ref_rows[j * R + t: j * R + t + 1], 0.6, 50, 0.95, [[u]])[0]
    dig = lcb._dev.u64_tensor(keys, DEV)
    cache.insert_batch(dig, torch.full((n,), R, dtype=torch.int32, device=DEV),
                       torch.full((n,), V, dtype=torch.int32, device=DEV), rows,
                       torch.arange(n, dtype=torch.int64, device=DEV) * R, torch.from_numpy(tok).to(DEV), R)
    for j in range(n):
        e = cache.lookup(lcb.StateKey(keys[j]))
        assert e is not None and len(e) == R
        assert np.array_equal(e.logits_seq, ref_rows[j * R:(j + 1) * R])
        assert e.token_seq == tok[j * R:(j + 1) * R].tolist()
    T = torch.full((n,), 0.6, dtype=torch.float64, device=DEV)
    K = torch.full((n,), 50, dtype=torch.int32, device=DEV)
    P = torch.full((n,), 0.95, dtype=torch.float64, device=DEV)
    rtok, rep, div, slot, ln = cache.replay_stepwise(dig, R, 1, lcb._dev.u64_tensor(seeds, DEV), T, K, P)
    assert np.all(slot.cpu().numpy() >= 0)
    assert np.all(rep.cpu().numpy() == R) and np.all(div.cpu().numpy() == -1)
    assert np.array_equal(rtok.cpu().numpy(), tok)


def test_cache_update_shape_errors_and_accounting():
    cache = lcb.LogitsCache()
    with pytest.raises(lcb.ConfigError):
        cache.update(lcb.StateKey.of([1]), np.zeros((5, 8), np.float32), [1, 2, 3])
    z = np.random.default_rng(0).normal(size=(500, 256)).astype(np.float32)
    e = cache.update(lcb.StateKey.of([1]), z, list(range(500)))
    assert e.nbytes == 500 * 256 * 4 + 500 * lcb.TOKEN_OVERHEAD_BYTES
    assert cache.total_bytes == e.nbytes
    got = cache.lookup(lcb.StateKey.of([1]))
    assert got.logits_seq.shape == (500, 256) and got.token_seq == list(range(500))
    assert np.array_equal(got.logits_seq, z)


def test_cache_narrow_then_wide_entries():
    cache = lcb.LogitsCache()
    cache.update(lcb.StateKey.of([1, 2]), np.ones((5, 32), np.float32), [0, 1, 2, 3, 4])
    cache.update(lcb.StateKey.of([3]), np.ones((2, 64), np.float32), [0, 1])
    a = cache.lookup(lcb.StateKey.of([1, 2]))
    assert a.vocab_size == 32 and a.logits_seq.shape == (5, 32) and np.all(a.logits_seq == 1)
    assert len(cache) == 2


def test_replay_stepwise_matches_oracle():
    """Fused lookup -> speculative step-wise resample -> acceptance vs the oracle."""
    V, n_req, L, nb = 2048, 6, 40, 5
    cache = lcb.LogitsCache(1 << 30, vocab=V, dtype="bfloat16", max_rows=64)
    prompts = [[r, 3, 5] for r in range(n_req)]
    keys = [mixing_ref.hash_tokens(p) for p in prompts]
    rows = mixing_ref.bf16_round(mixing_ref.fill_rows_np([mixing_ref.mix2(5, i) for i in range(n_req * L)], V, 2.5))
    cached_tok = np.random.default_rng(1).integers(0, V, n_req * L).astype(np.int32)
    # make early positions agree with the likely sample so replays run for a while
    cached_tok = np.where(np.arange(n_req * L) % L < 10, rows.argmax(1), cached_tok).astype(np.int32)
    lens = np.full(n_req, L, np.int32)
    lens[1] = 17
    offs = (np.arange(n_req) * L).astype(np.int64)
    cache.insert_batch(lcb._dev.u64_tensor(keys, DEV), torch.from_numpy(lens).to(DEV),
                       torch.full((n_req,), V, dtype=torch.int32, device=DEV),
                       torch.from_numpy(rows).to(DEV).to(torch.bfloat16), torch.from_numpy(offs).to(DEV),
                       torch.from_numpy(cached_tok).to(DEV), L)
    digests = lcb._dev.u64_tensor(keys + [12345], DEV)  # last request misses
    seeds = [mixing_ref.mix2(1, b) for b in range((n_req + 1) * nb)]
    T = torch.full((n_req + 1,), 0.6, dtype=torch.float64, device=DEV)
    K = torch.zeros(n_req + 1, dtype=torch.int32, device=DEV)
    Pp = torch.full((n_req + 1,), 0.9, dtype=torch.float64, device=DEV)
    tok, rep, div, slot, ln = cache.replay_stepwise(digests, 32, nb, lcb._dev.u64_tensor(seeds, DEV), T, K, Pp)
    rep = rep.cpu().numpy().reshape(n_req + 1, nb)
    for r in range(n_req):
        lim = min(int(lens[r]), 32)
        for b in range(nb):
            want_rep = 0
            for t in range(lim):
                u = mixing_ref.uniform(seeds[r * nb + b], t)
                y = _oracle_tokens(rows[r * L + t: r * L + t + 1], 0.6, None, 0.9, [[u]])[0]
                want_rep = t + 1
                if y != cached_tok[r * L + t]:
                    break
            assert rep[r, b] == want_rep, (r, b)
    assert np.all(rep[n_req] == 0)


def test_replay_hotspot_matches_oracle():
    """ReplayPolicy.HOTSPOT on the device (engine.py:311-326) vs the oracle loop: draws only at
    hotspots with draw number = hotspots before t, cached tokens copied elsewhere, stop after the
    first differing hotspot sample; tokens equal the engine's out list."""
    V, n_req, L, nb = 2048, 6, 40, 4
    cache = lcb.LogitsCache(1 << 30, vocab=V, dtype="bfloat16", max_rows=64)
    keys = [mixing_ref.hash_tokens([r, 9, 4]) for r in range(n_req)]
    rows = mixing_ref.bf16_round(mixing_ref.fill_rows_np([mixing_ref.mix2(6, i) for i in range(n_req * L)], V, 2.5))
    rng = np.random.default_rng(4)
    cached_tok = rng.integers(0, V, n_req * L).astype(np.int32)
    cached_tok = np.where(np.arange(n_req * L) % L < 12, rows.argmax(1), cached_tok).astype(np.int32)
    lens = np.full(n_req, L, np.int32)
    lens[2] = 9
    offs = (np.arange(n_req) * L).astype(np.int64)
    cache.insert_batch(lcb._dev.u64_tensor(keys, DEV), torch.from_numpy(lens).to(DEV),
                       torch.full((n_req,), V, dtype=torch.int32, device=DEV),
                       torch.from_numpy(rows).to(DEV).to(torch.bfloat16), torch.from_numpy(offs).to(DEV),
                       torch.from_numpy(cached_tok).to(DEV), L)
    hot = [tuple(sorted(rng.choice(L, int(rng.integers(0, 14)), replace=False).tolist())) for _ in range(n_req)]
    hot[0] = ()
    hot.append((1, 2))  # the missing request
    digests = lcb._dev.u64_tensor(keys + [777], DEV)
    seeds = [mixing_ref.mix2(2, b) for b in range((n_req + 1) * nb)]
    T = torch.full((n_req + 1,), 0.6, dtype=torch.float64, device=DEV)
    K = torch.zeros(n_req + 1, dtype=torch.int32, device=DEV)
    Pp = torch.full((n_req + 1,), 0.9, dtype=torch.float64, device=DEV)
    max_pos = 32
    tok, rep, div, slot, ln = cache.replay_hotspot(digests, max_pos, nb, lcb._dev.u64_tensor(seeds, DEV), T, K,
                                                   Pp, hot)
    tok, rep, div = tok.clone(), rep.clone(), div.clone()
    # compact task list (only hotspot positions become tasks): identical results
    d_di = cache.hotspot_draw_index(hot, max_pos, DEV)
    tl, rl, dl, _, _ = cache.replay_hotspot(digests, max_pos, nb, lcb._dev.u64_tensor(seeds, DEV), T, K, Pp,
                                            draw_index=d_di, hot_list=cache.hotspot_list(d_di))
    assert torch.equal(rl, rep) and torch.equal(dl, div)
    rep_np = rep.cpu().numpy().reshape(n_req + 1, nb)
    tk, tkl = tok.cpu().numpy().reshape(n_req + 1, max_pos, nb), tl.cpu().numpy().reshape(n_req + 1, max_pos, nb)
    for r in range(n_req + 1):
        for b in range(nb):
            n_out = int(rep_np[r, b])
            assert np.array_equal(tk[r, :n_out, b], tkl[r, :n_out, b])
    tok = tok.cpu().numpy().reshape(n_req + 1, max_pos, nb)
    rep = rep.cpu().numpy().reshape(n_req + 1, nb)
    div = div.cpu().numpy().reshape(n_req + 1, nb)
    for r in range(n_req):
        lim = min(int(lens[r]), max_pos)
        hs = set(hot[r])
        for b in range(nb):
            out, k, want_div = [], 0, -1
            for t in range(lim):
                yc = int(cached_tok[r * L + t])
                if t in hs:
                    u = mixing_ref.uniform(seeds[r * nb + b], k)
                    k += 1
                    y = _oracle_tokens(rows[r * L + t: r * L + t + 1], 0.6, None, 0.9, [[u]])[0]
                else:
                    y = yc
                out.append(y)
                if y != yc:
                    want_div = t
                    break
            assert rep[r, b] == len(out), (r, b)
            assert div[r, b] == want_div, (r, b)
            assert tok[r, :len(out), b].tolist() == out, (r, b)
    assert np.all(rep[n_req] == 0)


@pytest.mark.parametrize("conc,T,p,nd", [(2.5, 0.6, 0.9, 32), (0.0, 0.6, 0.9, 8), (2.5, 1.0, 0.5, 4),
                                         (5.0, 0.3, 0.99, 16), (1.0, 2.0, 0.95, 8)])
def test_staged_kernel_matches_oracle_and_other_tiers(conc, T, p, nd, monkeypatch):
    """The TMA-staged kernel (bf16, V <= 32768, top-p) against the oracle, and
    bit-identical to the row-warp path (LCB_NO_STAGE=1) on the same inputs."""
    V, n = 32000, 48
    rows = mixing_ref.bf16_round(mixing_ref.fill_rows_np([mixing_ref.mix2(23, i) for i in range(n)], V, conc))
    rng = np.random.default_rng(int(conc * 10 + T * 100 + p * 1000))
    ulists = [rng.random(nd) for _ in range(n)]
    tok, fl, cnt = _resample_rows(rows, T, None, p, ulists, dtype=torch.bfloat16)
    want = []
    for r in range(n):
        q = sampling_ref.truncate(sampling_ref.softmax(rows[r], T), None, p)
        want += [sampling_ref.draw(q, float(x)) for x in ulists[r]]
    assert tok.tolist() == want
    assert not np.any(fl & _capi.LC_DRAW_UNRESOLVED)
    monkeypatch.setenv("LCB_NO_STAGE", "1")
    tok2, _, _ = _resample_rows(rows, T, None, p, ulists, dtype=torch.bfloat16)
    assert tok2.tolist() == tok.tolist()


def _stage_rows_and_cases():
    """bf16 V=32000 rows that drive the staged kernel's less common branches."""
    V = 32000
    rng = np.random.default_rng(404)
    rows, cases = [], []
    base = mixing_ref.fill_rows_np([mixing_ref.mix2(31, i) for i in range(8)], V, 2.5)
    # all-negative rows (generic key path; max < 0)
    rows.append(base[0] - 20.0)
    # max in [0.5, 2]: histogram classes cross zero (generic key path)
    rows.append(base[1] * 0.2)
    # heavy ties at the cut: values from a small set
    rows.append(rng.choice(np.float32([3.0, 2.5, 2.0, 1.5, 1.0, 0.0, -1.0]), V).astype(np.float32))
    # flat row: huge nucleus
    rows.append(rng.uniform(-1, 1, V).astype(np.float32))
    # +-0 maximum (requeued to the CTA kernel)
    z = np.full(V, -3.0, np.float32)
    z[5], z[17] = -0.0, 0.0
    rows.append(z)
    # a peak plus a dense shoulder
    z = base[2].copy()
    z[100:400] = 14.0
    rows.append(z)
    return mixing_ref.bf16_round(np.stack(rows)), V


@pytest.mark.parametrize("T,p,nd", [(0.6, 0.9, 32), (1.0, 0.5, 8), (0.3, 0.999, 16), (0.0, 0.9, 4),
                                    (0.8, 0.9, 100)])
def test_staged_kernel_edge_rows(T, p, nd):
    """Staged-kernel branches (negative / zero-crossing maxima, ties at the cut,
    flat rows, signed-zero maxima, greedy rows, more draws than it keeps)
    against the oracle, and bit-identical to the row-warp path."""
    rows, V = _stage_rows_and_cases()
    rng = np.random.default_rng(int(T * 1000 + p * 100 + nd))
    ulists = [rng.random(nd) for _ in range(len(rows))]
    tok, fl, _ = _resample_rows(rows, T, None, p, ulists, dtype=torch.bfloat16)
    want = []
    for r in range(len(rows)):
        q = sampling_ref.truncate(sampling_ref.softmax(rows[r], T), None, p)
        want += [sampling_ref.draw(q, float(x)) for x in ulists[r]]
    assert tok.tolist() == want
    assert not np.any(fl & _capi.LC_DRAW_UNRESOLVED)


def test_staged_kernel_writes_every_draw_under_load():
    """A launch large enough to keep every group of every SM busy: every draw
    is written (no task lost between the producer FIFO, the stages and the
    requeue path) and a sample of rows matches the oracle."""
    V, n, nd = 32000, 4096, 32
    states = lcb._dev.u64_tensor([mixing_ref.mix2(77, i) for i in range(n)], DEV)
    rows = torch.empty((n, V), dtype=torch.bfloat16, device=DEV)
    _capi.check(_capi.lib.lc_fill_logits(states.data_ptr(), n, V, 2.5, 5.0, _capi.LC_BF16, rows.data_ptr(), V,
                                         None))
    tasks = lcb.make_tasks(row=np.arange(n), temperature=0.6, top_p=0.9, draw_begin=np.arange(n) * nd,
                           draw_end=np.arange(n) * nd + nd)
    u = np.random.default_rng(5).random(n * nd)
    ud = torch.from_numpy(u).to(DEV)
    for _ in range(3):
        tok = torch.full((n * nd,), -7, dtype=torch.int32, device=DEV)
        fl = torch.zeros(n * nd, dtype=torch.uint8, device=DEV)
        lcb.resample(rows, tasks, u=ud, out=(tok, fl))
        got = tok.cpu().numpy()
        assert not np.any(got == -7)
    host = rows.float().cpu().numpy()
    for r in range(0, n, 97):
        q = sampling_ref.truncate(sampling_ref.softmax(host[r], 0.6), None, 0.9)
        assert got[r * nd:(r + 1) * nd].tolist() == [sampling_ref.draw(q, float(x)) for x in u[r * nd:(r + 1) * nd]]


@pytest.mark.parametrize("V,conc,T,k,p,nd", [(151936, 2.5, 0.6, 50, 0.95, 1), (151936, 0.0, 1.0, 50, 0.95, 4),
                                             (128256, 2.5, 0.6, 20, 0.9, 8), (151936, 2.5, 0.0, 50, 0.95, 2),
                                             (40000, 1.0, 0.8, 64, 1.0, 3), (151936, 5.0, 0.3, 1, 0.5, 2)])
def test_wide_kernel_matches_oracle_and_cta_kernel(V, conc, T, k, p, nd, monkeypatch):
    """The TMA-staged top-k kernel (bf16 rows wider than 32000 ids) against the
    oracle, and bit-identical to the CTA kernel (LCB_NO_STAGE=1)."""
    n = 24
    rows = mixing_ref.bf16_round(mixing_ref.fill_rows_np([mixing_ref.mix2(29, i) for i in range(n)], V, conc))
    rng = np.random.default_rng(int(V + conc * 10 + T * 100 + k))
    ulists = [rng.random(nd) for _ in range(n)]
    tok, fl, cnt = _resample_rows(rows, T, k, p, ulists, dtype=torch.bfloat16)
    want = []
    for r in range(n):
        q = sampling_ref.truncate(sampling_ref.softmax(rows[r], T), k, p)
        want += [sampling_ref.draw(q, float(x)) for x in ulists[r]]
    assert tok.tolist() == want
    assert not np.any(fl & _capi.LC_DRAW_UNRESOLVED)
    monkeypatch.setenv("LCB_NO_STAGE", "1")
    tok2, _, _ = _resample_rows(rows, T, k, p, ulists, dtype=torch.bfloat16)
    assert tok2.tolist() == tok.tolist()


@pytest.mark.parametrize("window", [1, 3, 8, 64])
def test_replay_windowed_equals_full_replay(window):
    """Windowed step-wise replay (rows resampled only while a branch is live) gives the full
    replay's replayed_len / diverged_at and the same tokens at every accepted position."""
    V, n_req, L, nb, max_pos = 4096, 9, 40, 6, 32
    cache = lcb.LogitsCache(1 << 30, vocab=V, dtype="bfloat16", max_rows=64)
    keys = [mixing_ref.hash_tokens([r, 7, 1]) for r in range(n_req)]
    rows = mixing_ref.bf16_round(mixing_ref.fill_rows_np([mixing_ref.mix2(9, i) for i in range(n_req * L)], V, 2.5))
    rng = np.random.default_rng(4)
    cached_tok = rng.integers(0, V, n_req * L).astype(np.int32)
    # agree with the argmax for a request-dependent prefix so replays end at different windows
    agree = np.arange(n_req * L) % L < (np.arange(n_req * L) // L) * 3
    cached_tok = np.where(agree, rows.argmax(1), cached_tok).astype(np.int32)
    lens = np.full(n_req, L, np.int32)
    lens[2] = 5
    lens[4] = 1
    offs = (np.arange(n_req) * L).astype(np.int64)
    cache.insert_batch(lcb._dev.u64_tensor(keys, DEV), torch.from_numpy(lens).to(DEV),
                       torch.full((n_req,), V, dtype=torch.int32, device=DEV),
                       torch.from_numpy(rows).to(DEV).to(torch.bfloat16), torch.from_numpy(offs).to(DEV),
                       torch.from_numpy(cached_tok).to(DEV), L)
    digests = lcb._dev.u64_tensor(keys + [999], DEV)  # the last request misses
    n = n_req + 1
    seeds = lcb._dev.u64_tensor([mixing_ref.mix2(3, b) for b in range(n * nb)], DEV)
    T = torch.full((n,), 0.6, dtype=torch.float64, device=DEV)
    K = torch.zeros(n, dtype=torch.int32, device=DEV)
    Pp = torch.full((n,), 0.9, dtype=torch.float64, device=DEV)
    tok_f, rep_f, div_f, slot, ln = cache.replay_stepwise(digests, max_pos, nb, seeds, T, K, Pp)
    tok_f, rep_f, div_f = tok_f.clone(), rep_f.clone(), div_f.clone()
    s2, g2, l2, v2 = cache.lookup_batch(digests)
    tok_w, rep_w, div_w, nwin = cache.replay_windowed(s2, g2, l2, v2, max_pos, nb, seeds, T, K, Pp, window=window)
    assert torch.equal(rep_w, rep_f) and torch.equal(div_w, div_f)
    rep = rep_f.cpu().numpy().reshape(n, nb)
    tf = tok_f.cpu().numpy().reshape(n, max_pos, nb)
    tw = tok_w.cpu().numpy().reshape(n, max_pos, nb)
    for r in range(n):
        for b in range(nb):
            assert np.array_equal(tf[r, : rep[r, b], b], tw[r, : rep[r, b], b]), (r, b)
    assert nwin <= -(-max_pos // window)
    assert rep.max() > window or window >= max_pos  # some replay crosses a window boundary


@pytest.mark.parametrize("V", [5, 1000, 32000, 151936])
def test_draw_probs_block_parallel_matches_oracle(V):
    """lc_draw_probs (block-parallel pairwise total, scanned chunk sums, certified crossing with the
    sequential fallback) vs numpy's searchsorted(cumsum(q), u*q.sum(), 'right'), including targets
    placed exactly on cumsum values and zero-probability runs."""
    rng = np.random.default_rng(V)
    q = rng.random(V) ** 4
    q[rng.random(V) < 0.3] = 0.0
    q[-3:] = 0.0
    q /= q.sum()
    cdf = np.cumsum(q)
    tot = q.sum()
    us = list(rng.random(300)) + [0.0, 1.0 - 2 ** -53]
    us += [float(cdf[i] / tot) for i in rng.integers(0, V, 40)]  # targets on (or next to) a cdf value
    n = len(us)
    d = DEV
    p = torch.from_numpy(q).to(d).reshape(1, V).expand(n, V).contiguous()
    ut = torch.tensor(us, dtype=torch.float64, device=d)
    tok = torch.empty(n, dtype=torch.int32, device=d)
    fl = torch.empty(n, dtype=torch.uint8, device=d)
    _capi.check(_capi.lib.lc_draw_probs(p.data_ptr(), V, n, V, ut.data_ptr(), tok.data_ptr(), fl.data_ptr(),
                                        lcb._dev.stream_ptr(d)), "lc_draw_probs")
    want = [sampling_ref.draw(q, u) for u in us]
    assert tok.cpu().tolist() == want


def test_prob_stats_match_numpy():
    rng = np.random.default_rng(3)
    for V in (2, 17, 32000):
        p = rng.random(V)
        p[rng.random(V) < 0.2] = 0.0
        p /= p.sum()
        nz = p[p > 0]
        assert abs(lcb.entropy(p) - float(-(nz * np.log(nz)).sum())) < 1e-12 * max(1.0, np.log(V))
        assert lcb.max_prob(p) == float(p.max())


def test_rowwarp_untruncated_draw_regression_c1():
    """C1 bench check leg, round 2: row 10479 (state mix2(7, 10479)), seed mix2(137, 20), draw
    number 479 -> numpy 23235 (margins ~2e-8 of the mass on both sides), the row-warp FAST tier
    returned 23236: its correlated bound ignored that inside the hit segment the walk sums its own
    exponentials, not the fused pass's (which produced the segment prefixes and K)."""
    V = 32000
    row = mixing_ref.fill_rows_np([mixing_ref.mix2(7, 10479)], V, 2.5)
    u = float(mixing_ref.uniforms_np(np.array([mixing_ref.mix2(137, 20)], dtype=np.uint64), np.array([479]))[0])
    tok, fl, _ = _resample_rows(row, 0.6, None, 1.0, [[u]])
    assert tok.tolist() == _oracle_tokens(row, 0.6, None, 1.0, [[u]]) == [23235]


@pytest.mark.parametrize("V,conc,T", [(32000, 2.5, 0.6), (32000, 0.0, 1.0), (32000, 2.5, 1.3),
                                       (128256, 2.5, 0.6), (128256, 0.0, 1.0)])
def test_untruncated_targets_near_cdf_boundaries(V, conc, T):
    """Untruncated fp32 rows (C1 shape): targets placed within 1e-9 .. 1e-6 of the mass from a cdf
    boundary, at every depth of the row (segment starts, inside segments, u -> 1), on both sides;
    every token must equal numpy's searchsorted(cumsum(p), u * p.sum(), 'right')."""
    nrows = 12 if V <= 32000 else 6  # (V > 65536: the CTA kernel)
    rng = np.random.default_rng(int(conc * 10 + T * 100) + V)
    rows = mixing_ref.fill_rows_np([mixing_ref.mix2(11, 777 + i) for i in range(nrows)], V, conc)
    ulists = []
    for z in rows:
        p = sampling_ref.softmax(z, T)
        cdf = np.cumsum(p) / p.sum()
        js = np.concatenate([rng.integers(0, V - 1, 40), np.arange(2047, V - 1, 2048)[:8], [V - 2, V // 2]])
        us = []
        for j in js:
            for rel in (1e-9, 1e-8, 1e-7, 1e-6):
                for sgn in (-1.0, 1.0):
                    x = cdf[j] + sgn * rel
                    if 0.0 <= x < 1.0:
                        us.append(float(x))
        ulists.append(us)
    tok, fl, cnt = _resample_rows(rows, T, None, 1.0, ulists)
    assert tok.tolist() == _oracle_tokens(rows, T, None, 1.0, ulists)
    assert not np.any(fl & _capi.LC_DRAW_UNRESOLVED)


@pytest.mark.parametrize("dtype", ["float32", "bfloat16"])
def test_resample_entropy_epilogue_matches_oracle(dtype):
    """lc_draws.d_entropy / d_pmax: per task, -sum p ln p and max p of softmax(z, T) over the task's
    row (sampling.py:112-119), for explicit rows and for cached rows (slot, pos)."""
    V, n = 32000, 24
    rows = mixing_ref.fill_rows_np([mixing_ref.mix2(21, i) for i in range(n)], V, 2.5)
    if dtype == "bfloat16":
        rows = mixing_ref.bf16_round(rows)
    Ts = [0.6, 1.0, 0.0, 1.7] * (n // 4)
    tasks = lcb.make_tasks(row=np.arange(n), temperature=np.array(Ts), top_p=0.9, draw_begin=np.arange(n),
                           draw_end=np.arange(n) + 1)
    z = torch.from_numpy(rows).to(DEV).to(getattr(torch, dtype))
    H = torch.empty(n, dtype=torch.float64, device=DEV)
    P = torch.empty(n, dtype=torch.float64, device=DEV)
    u = torch.full((n,), 0.5, dtype=torch.float64, device=DEV)
    lcb.resample(z, tasks, u=u, entropy=H, pmax=P)
    for i in range(n):
        p = sampling_ref.softmax(rows[i], Ts[i])
        nz = p[p > 0]
        assert abs(H[i].item() - float(-(nz * np.log(nz)).sum())) <= 1e-11 * max(1.0, float(np.log(V)))
        assert abs(P[i].item() - float(p.max())) <= 1e-12


@pytest.mark.parametrize("V,conc,T,k,p", [(32000, 2.5, 0.6, None, 0.9), (32000, 0.0, 1.0, None, 0.9),
                                         (151936, 2.5, 0.6, 50, 0.95), (32000, 2.5, 0.6, 7, 1.0),
                                         (1000, 0.0, 5.0, None, 0.5), (128256, 0.0, 0.6, None, 0.99)])
def test_truncate_probs_fast_path_matches_oracle(V, conc, T, k, p):
    """lc_truncate_probs (radix-select fast path; rows with > 4096 kept values or an unreachable
    target take the slow path) vs numpy truncate(softmax(z, T), k, p), bit for bit, including
    rows with many equal probabilities (quantised logits)."""
    rng = np.random.default_rng(V + int(T * 10))
    rows = mixing_ref.fill_rows_np([mixing_ref.mix2(31, i) for i in range(4)], V, conc)
    rows[3] = np.round(rows[3] * 2) / 2  # ties
    for z in rows:
        prob = sampling_ref.softmax(z, T)
        want = sampling_ref.truncate(prob, k, p)
        got = lcb.truncate(prob, k, p)
        assert np.array_equal(np.asarray(got), want), (V, k, p)
    assert rng is not None
