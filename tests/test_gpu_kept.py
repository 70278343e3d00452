"""Kept sets of the fused resample kernels vs the reference (sampling.py:71-94).

North star: "top-k index sets ... must be bit-exact".  Every fused kernel
(staged bf16 nucleus kernel, wide top-k kernel, row-warp kernel, CTA kernel,
EXACT tier) reports each task's kept-set size K (``lc_draws.d_kept``); the set
is the first K ids in (logit desc, id asc) order, checked against the golden
``kept`` arrays the reference produced (tests/golden/sampling.npz, 881 cases)
and against the oracle at the configs' vocabularies.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import mixing_ref, sampling_ref
from tests.golden_io import sampling_cases
from tests.kept_check import kept_mismatch, zorder_prefix

pytestmark = pytest.mark.gpu

lcb = pytest.importorskip("paper_2604_17353_b200")
from paper_2604_17353_b200 import _capi  # noqa: E402

DEV = torch.device("cuda", 0)


def _resample_kept(rows, T, k, p, u_lists, dtype=torch.float32):
    z = torch.from_numpy(np.ascontiguousarray(rows, dtype=np.float32)).to(DEV).to(dtype)
    n = len(rows)
    counts = np.array([len(x) for x in u_lists])
    begin = np.concatenate([[0], np.cumsum(counts)[:-1]])
    tasks = lcb.make_tasks(row=np.arange(n), temperature=T, top_k=k, top_p=p, draw_begin=begin,
                           draw_end=begin + counts)
    u = torch.tensor(np.concatenate(u_lists), dtype=torch.float64, device=DEV)
    kept = torch.full((n,), -7, dtype=torch.int32, device=DEV)
    tok, fl = lcb.resample(z, tasks, u=u, kept=kept)
    return tok.cpu().numpy(), kept.cpu().numpy()


def test_zorder_prefix_helper():
    z = np.array([1.0, 3.0, 3.0, -np.inf, 2.0, 3.0], np.float32)
    assert zorder_prefix(z, 4).tolist() == [1, 2, 5, 4]
    assert zorder_prefix(z, 6).tolist() == [1, 2, 5, 4, 0, 3]


@pytest.mark.parametrize("as_bf16", [False, True])
def test_kept_sets_golden(as_bf16):
    """All reference golden cases: K == len(kept_order) and the kept ids == the golden set."""
    cases = sampling_cases()
    if as_bf16:
        cases = [c for c in cases if c.name.startswith("bf16_")]
    n = 0
    for c in cases:
        tok, kept = _resample_kept(c.z[None, :], c.T, c.top_k, c.top_p, [c.u],
                                   dtype=torch.bfloat16 if as_bf16 else torch.float32)
        assert tok.tolist() == c.tokens.tolist(), c.name
        p = sampling_ref.softmax(c.z, c.T)
        why = kept_mismatch(c.z, c.T, c.top_k, c.top_p, kept[0], p)
        assert why is None, (c.name, c.T, c.top_k, c.top_p, why)
        # the golden kept array itself (made by the reference, not by the oracle)
        got = zorder_prefix(c.z, int(kept[0]))
        assert np.array_equal(np.sort(got[p[got] > 0]), c.kept), c.name
        n += 1
    assert n > (100 if as_bf16 else 800)


@pytest.mark.parametrize("tier", ["precise", "exact"])
def test_kept_sets_forced_tiers(tier, monkeypatch):
    monkeypatch.setenv("LCB_FORCE_TIER", tier)
    for c in [c for c in sampling_cases() if len(c.z) <= 4099]:
        tok, kept = _resample_kept(c.z[None, :], c.T, c.top_k, c.top_p, [c.u])
        p = sampling_ref.softmax(c.z, c.T)
        got = zorder_prefix(c.z, int(kept[0]))
        assert np.array_equal(np.sort(got[p[got] > 0]), c.kept), (tier, c.name)


@pytest.mark.parametrize("V,conc,T,k,p,bf16,nrows", [
    (32000, 2.5, 0.6, None, 0.9, True, 256),     # C2 (staged kernel)
    (32000, 0.0, 0.6, None, 0.9, True, 96),      # flat: large nuclei (staged kernel)
    (32000, 2.5, 1.0, None, 0.5, True, 96),
    (32000, 2.5, 0.6, None, 1.0, False, 64),     # C1 (row-warp kernel, untruncated: K = V)
    (32000, 0.0, 0.8, None, 0.95, False, 64),    # row-warp big nucleus
    (151936, 2.5, 0.6, 50, 0.95, True, 96),      # C3 / C5 (wide kernel)
    (151936, 0.0, 1.0, 50, 0.95, True, 32),
    (151936, 2.5, 0.6, 50, 0.95, False, 32),     # CTA kernel (fp32 top-k)
    (128256, 2.5, 0.6, None, 0.9, True, 32),     # wide rows, nucleus only (CTA kernel)
    (4099, 1.0, 0.25, 3, 0.999, False, 32),
])
def test_kept_sets_match_oracle_at_config_vocab(V, conc, T, k, p, bf16, nrows):
    states = [mixing_ref.mix2(31, V + i) for i in range(nrows)]
    rows = mixing_ref.fill_rows_np(states, V, conc)
    if bf16:
        rows = mixing_ref.bf16_round(rows)
    rng = np.random.default_rng(V + nrows)
    ul = [rng.random(4).tolist() for _ in range(nrows)]
    tok, kept = _resample_kept(rows, T, k, p, ul, dtype=torch.bfloat16 if bf16 else torch.float32)
    bad = []
    want_tok = []
    for i, z in enumerate(rows):
        prob = sampling_ref.softmax(z, T)
        why = kept_mismatch(z, T, k, p, kept[i], prob)
        if why:
            bad.append((i, why))
        q = sampling_ref.truncate(prob, k, p)
        want_tok += [sampling_ref.draw(q, float(u)) for u in ul[i]]
    assert not bad, bad[:5]
    assert tok.tolist() == want_tok


def test_kept_staged_vs_rowwarp_every_row(monkeypatch):
    """2,048 C2-shape rows: the staged kernel and the row-warp path (LCB_NO_STAGE=1) report the
    same kept count for every row and the same token for every draw."""
    V, n = 32000, 2048
    rows = mixing_ref.bf16_round(mixing_ref.fill_rows_np([mixing_ref.mix2(41, i) for i in range(n)], V, 2.5))
    rng = np.random.default_rng(3)
    ul = [rng.random(8).tolist() for _ in range(n)]
    tok_s, kept_s = _resample_kept(rows, 0.6, None, 0.9, ul, dtype=torch.bfloat16)
    monkeypatch.setenv("LCB_NO_STAGE", "1")
    tok_r, kept_r = _resample_kept(rows, 0.6, None, 0.9, ul, dtype=torch.bfloat16)
    assert np.array_equal(kept_s, kept_r)
    assert np.array_equal(tok_s, tok_r)
    assert (kept_s > 1).sum() > 300  # both nucleus regimes exercised
    # spot-check a sample against the oracle
    for i in range(0, n, 97):
        assert kept_mismatch(rows[i], 0.6, None, 0.9, kept_s[i]) is None, i


def test_kept_greedy_and_bad_rows():
    z = np.array([[1.0, np.nan, 0.0, 2.0], [5.0, 5.0, 1.0, -1.0], [5.0, 5.0, 1.0, -1.0],
                  [5.0, 5.0, 1.0, -1.0]], dtype=np.float32)
    for (T, k, p), want in (((0.0, None, 0.9), 1), ((0.0, 2, 1.0), 2), ((0.0, None, 1.0), 4)):
        tok, kept = _resample_kept(z, T, k, p, [[0.5]] * 4)
        assert kept[0] == -1 and tok[0] == -1
        assert kept[1:].tolist() == [want] * 3, (T, k, p)
        for i in range(1, 4):
            assert kept_mismatch(z[i], T, k, p, kept[i]) is None
