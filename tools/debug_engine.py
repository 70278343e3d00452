import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2604_17353_b200 as lcb
from paper_2604_17353_b200.engine import GenerateRequest, ModelConfig, WaveEngine
from tests.golden_io import load_json
sc = [s for s in load_json("engine_traces.json") if s["name"] == "stepwise_v64"][0]
seed, V, conc, rng = sc["model"]
eng = WaveEngine(ModelConfig(seed=seed, vocab_size=V, concentration=conc, logit_range=rng), 1 << 30, max_tokens=24,
                 device=torch.device("cuda", 0))
eng.register_agent("a")
wave = sc["waves"][0]
reqs = [GenerateRequest("a", pr, lcb.SamplingConfig(temperature=sc["T"], max_tokens=24, seed=r["seed"]),
                        lcb.ReplayPolicy.STEP_WISE) for pr, r in zip(sc["prompts"], wave)]
got = eng.generate_wave(reqs)
for i, (g, pr) in enumerate(zip(got, sc["prompts"])):
    e = eng.cache.lookup(lcb.StateKey.of(pr))
    ts = e.token_seq
    bad = [t for t in range(24) if ts[t] != g.tokens[t]]
    print(i, "slot", e.slot, "gen", e.gen, "len", len(e), "bad", bad, ts[:12], g.tokens[:12])
