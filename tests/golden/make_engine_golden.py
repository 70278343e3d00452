"""Engine traces from the REFERENCE ``InferenceEngine`` (test infrastructure).

Run in the build container (where ``/root/reference`` exists):

    cp -r /root/reference/pkg build/ref && (cd build/ref && python setup.py build_ext --inplace)
    PYTHONPATH=build/ref/src python tests/golden/make_engine_golden.py

Each scenario is a model config plus WAVES of requests with distinct prompt keys;
the reference engine runs every request of a wave in order, wave after wave (the
order ``paper_2604_17353_b200.engine.WaveEngine`` defines).  Recorded per request:
tokens and ReplayOutcome (engine.py:364-371) plus the pass counters; after the
last wave, every cached entry: length, token_seq, and a SHA-1 of its float32
logits rows (the write-back rows, engine.py:349-361, bit-exact).
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = os.environ.get("AGENTSERVE_SRC", os.path.join(HERE, "..", "..", "build", "ref", "src"))
sys.path.insert(0, REF)

from agentserve.engine import GenerateRequest, InferenceEngine  # noqa: E402
from agentserve.logits_cache import ReplayPolicy  # noqa: E402
from agentserve.mixing import RngStream, mix2  # noqa: E402
from agentserve.model import ModelConfig  # noqa: E402
from agentserve.sampling import HotspotParams, SamplingConfig  # noqa: E402


def prompts_for(seed, n, vocab, lo=4, hi=14):
    s = RngStream(seed)
    out = []
    for _ in range(n):
        k = lo + int(s.next_float() * (hi - lo))
        out.append([int(s.next_float() * vocab) for _ in range(k)])
    return out


SCENARIOS = [
    # name, model (seed, vocab, conc, range), policy, sampling (T, top_k, top_p), prompts, siblings, max_tokens
    dict(name="stepwise_v64", model=(11, 64, 2.0, 5.0), policy="step_wise", T=0.8, k=None, p=1.0, n=6, sib=4, L=24),
    dict(name="stepwise_v64_cold_T", model=(11, 64, 2.0, 5.0), policy="step_wise", T=0.3, k=None, p=1.0, n=5,
         sib=3, L=30),
    dict(name="hotspot_v64", model=(5, 64, 2.0, 5.0), policy="hotspot", T=1.0, k=None, p=1.0, n=6, sib=4, L=24,
         hp=(0.01, 0.6, None)),
    dict(name="hotspot_v256_cap", model=(9, 256, 1.5, 5.0), policy="hotspot", T=0.9, k=None, p=0.95, n=4, sib=3,
         L=32, hp=(0.001, 0.5, 4)),
    dict(name="none_v128", model=(3, 128, 2.0, 5.0), policy="none", T=1.0, k=None, p=1.0, n=4, sib=2, L=20),
    dict(name="topk_topp_v512", model=(21, 512, 2.5, 5.0), policy="step_wise", T=1.0, k=20, p=0.9, n=5, sib=3,
         L=40),
    dict(name="greedy_v64", model=(5, 64, 2.0, 5.0), policy="step_wise", T=0.0, k=None, p=1.0, n=3, sib=3, L=16),
    dict(name="stepwise_v32000_topp", model=(7, 32000, 2.5, 5.0), policy="step_wise", T=0.6, k=None, p=0.9, n=3,
         sib=3, L=12),
    dict(name="grow_v64", model=(13, 64, 2.0, 5.0), policy="step_wise", T=0.5, k=None, p=1.0, n=4, sib=3,
         L=[8, 20, 12]),
]


def run(sc):
    seed, V, conc, rng = sc["model"]
    hp = HotspotParams(*sc["hp"]) if "hp" in sc else HotspotParams()
    eng = InferenceEngine(ModelConfig(seed=seed, vocab_size=V, concentration=conc, logit_range=rng),
                          capacity_tokens=1_000_000, logits_budget_bytes=1 << 30, hotspot_params=hp)
    eng.register_agent("a")
    pol = {"step_wise": ReplayPolicy.STEP_WISE, "hotspot": ReplayPolicy.HOTSPOT, "none": ReplayPolicy.NONE}[sc["policy"]]
    prompts = prompts_for(mix2(seed, 77), sc["n"], V)
    Ls = sc["L"] if isinstance(sc["L"], list) else [sc["L"]] * sc["sib"]
    waves = []
    for w in range(sc["sib"]):
        res = []
        for i, pr in enumerate(prompts):
            cfg = SamplingConfig(temperature=sc["T"], top_k=sc["k"], top_p=sc["p"], max_tokens=Ls[w],
                                 seed=mix2(seed, 1000 * w + i))
            r = eng.generate(GenerateRequest("a", list(pr), cfg, pol, request_id=f"w{w}r{i}"))
            o = r.outcome
            res.append(dict(tokens=r.tokens, replayed_len=o.replayed_len, diverged_at=o.diverged_at,
                            total_len=o.total_len, forward_passes_saved=o.forward_passes_saved,
                            was_revisit=r.was_revisit, prefill_passes=r.prefill_passes,
                            decode_passes=r.decode_passes, prefill_input=r.prefill_input, seed=cfg.seed,
                            max_tokens=cfg.max_tokens))
        waves.append(res)
    entries = {}
    for d, e in eng.cache.entries.items():
        rows = np.ascontiguousarray(e.logits_seq, dtype=np.float32)
        entries[str(d)] = dict(n=len(e), tokens=list(e.token_seq), sha1=hashlib.sha1(rows.tobytes()).hexdigest())
    return dict(sc, prompts=prompts, waves=waves, entries=entries, total_bytes=eng.cache.total_bytes,
                lookups=eng.cache.lookups, hits=eng.cache.hits)


def main():
    out = [run(sc) for sc in SCENARIOS]
    with open(os.path.join(HERE, "engine_traces.json"), "w") as f:
        json.dump(out, f)
    for o in out:
        reps = [r["replayed_len"] for w in o["waves"] for r in w]
        print(o["name"], "replayed", sum(reps), "entries", len(o["entries"]))


if __name__ == "__main__":
    main()
