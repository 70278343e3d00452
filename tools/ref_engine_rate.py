"""Tokens/s of the reference's own InferenceEngine.generate on the bench_engine.py workload shape
(BUILD CONTAINER ONLY: imports the reference from /root/reference, which the GPU box does not
have).  One core, AGENTSERVE_PURE=1 (numpy producer), W requests x L tokens, a cold wave then a
revisit wave with new seeds (ReplayPolicy.STEP_WISE).

AGENTSERVE_PURE=1 python tools/ref_engine_rate.py [W] [L]
"""
import sys
import time

sys.path.insert(0, "/root/reference/pkg/src")
from agentserve.engine import GenerateRequest, InferenceEngine  # noqa: E402
from agentserve.logits_cache import ReplayPolicy  # noqa: E402
from agentserve.model import ModelConfig  # noqa: E402
from agentserve.sampling import SamplingConfig  # noqa: E402

V = 32000
W = int(sys.argv[1]) if len(sys.argv) > 1 else 8
L = int(sys.argv[2]) if len(sys.argv) > 2 else 128
model = ModelConfig(seed=7, vocab_size=V, concentration=2.5, logit_range=5.0)
eng = InferenceEngine(model, logits_budget_bytes=4 * W * L * (V * 4 + 8))
eng.register_agent("a")
prompts = [[1 + (r % 251), 2 + (r // 251) % 251] + [(r * 31 + i) % 1000 for i in range(40)] for r in range(W)]


def wave(k):
    return [GenerateRequest("a", p, SamplingConfig(temperature=0.6, top_p=0.9, max_tokens=L, seed=k * 1_000_003 + r),
                            ReplayPolicy.STEP_WISE, request_id=f"{k}-{r}") for r, p in enumerate(prompts)]


t = time.perf_counter()
res = [eng.generate(q) for q in wave(1)]
cold = time.perf_counter() - t
t = time.perf_counter()
res2 = [eng.generate(q) for q in wave(2)]
rev = time.perf_counter() - t
print({"cold_tokens_per_s": sum(len(r.tokens) for r in res) / cold,
       "revisit_tokens_per_s": sum(len(r.tokens) for r in res2) / rev,
       "replayed": sum(r.outcome.replayed_len for r in res2), "cores": 1})
