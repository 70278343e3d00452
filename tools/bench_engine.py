"""Wave-engine throughput: InferenceEngine._generate (engine.py:270-388) for
waves of requests on the device (paper_2604_17353_b200.engine.WaveEngine.generate_wave).

Workload: a C2-shaped model (V = 32000, concentration 2.5, range 5.0, bf16 cache), W requests per
wave with distinct prompts, max_tokens L, T 0.6 + top-p 0.9, ReplayPolicy.STEP_WISE.  Wave 1 is
cold (every request misses: prefill row + L - 1 decode rows produced into the slab, one resample
launch per decode step); wave 2 repeats the prompts with new seeds (lookup hits, step-wise replay
of the cached trajectories, the miss path from the divergence on, write-back keeping the replayed
prefix in place).  Prints one JSON line: generated tokens/s of each wave kind (CUDA events,
host synchronisation inside generate_wave included: this is the public call a server makes).

python tools/bench_engine.py [--requests 256] [--tokens 128] [--waves 3]
"""

from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--requests", type=int, default=256)
    ap.add_argument("--tokens", type=int, default=128)
    ap.add_argument("--waves", type=int, default=3)
    ap.add_argument("--vocab", type=int, default=32000)
    a = ap.parse_args()

    import torch

    from paper_2604_17353_b200 import ReplayPolicy, SamplingConfig
    from paper_2604_17353_b200.engine import GenerateRequest, ModelConfig, WaveEngine

    dev = torch.device("cuda", 0)
    W, L, V = a.requests, a.tokens, a.vocab
    model = ModelConfig(seed=7, vocab_size=V, concentration=2.5, logit_range=5.0)
    budget = 4 * W * L * (V * 4 + 8)  # room for every trajectory: no eviction during the run
    eng = WaveEngine(model, budget, dtype="bfloat16", max_tokens=L, key_capacity=4 * W + 64, device=dev)
    eng.register_agent("a")
    prompts = [[1 + (r % 251), 2 + (r // 251) % 251] + [(r * 31 + i) % 1000 for i in range(40)] for r in range(W)]

    def wave(seed_base):
        return [GenerateRequest("a", p, SamplingConfig(temperature=0.6, top_p=0.9, max_tokens=L,
                                                       seed=seed_base * 1_000_003 + r),
                                ReplayPolicy.STEP_WISE, request_id=f"{seed_base}-{r}") for r, p in enumerate(prompts)]

    def timed(reqs):
        torch.cuda.synchronize(dev)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        res = eng.generate_wave(reqs)
        e.record()
        torch.cuda.synchronize(dev)
        return res, s.elapsed_time(e)

    # warm-up on other prompts (kernels, allocations), then a fresh engine state for the timed waves
    timed(wave(999)[: min(W, 32)])
    cold_ms, cold_tok, rev_ms, rev_tok, replayed, decoded = 0.0, 0, 0.0, 0, 0, 0
    for k in range(a.waves):
        if k == 0:
            res, ms = timed(wave(1))
            cold_ms += ms
            cold_tok += sum(len(r.tokens) for r in res)
        else:
            res, ms = timed(wave(1 + k))
            rev_ms += ms
            rev_tok += sum(len(r.tokens) for r in res)
            replayed += sum(r.outcome.replayed_len for r in res)
            decoded += sum(r.decode_passes for r in res)
    line = {
        "metric": "engine_generated_tokens_per_s",
        "workload": f"WaveEngine.generate_wave, {W} requests x {L} tokens per wave, V={V} bf16 cache, "
                    "T 0.6 + top-p 0.9, ReplayPolicy.STEP_WISE",
        "cold_wave": {"tokens": cold_tok, "ms": cold_ms, "tokens_per_s": cold_tok / (cold_ms * 1e-3)},
        "revisit_waves": {"waves": a.waves - 1, "tokens": rev_tok, "ms": rev_ms,
                          "tokens_per_s": rev_tok / (rev_ms * 1e-3) if rev_ms else None,
                          "replayed_tokens": replayed, "decode_passes": decoded,
                          "position_hit_ratio": replayed / rev_tok if rev_tok else None},
        "forward_passes": {"prefill": eng.cost.prefill_passes, "decode": eng.cost.decode_passes},
        "decode_loop": "one CUDA graph per wave" if os.environ.get("LCB_ENGINE_GRAPH", "0") == "1" else "eager launches",
        "note": "synthetic model (the reference producer), one device; timings include generate_wave's host "
                "synchronisation and result lists (the public call)",
    }
    print(json.dumps(line))


if __name__ == "__main__":
    main()
