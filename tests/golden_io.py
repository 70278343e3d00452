"""Loaders for the committed golden vectors (tests/golden/*, made by make_golden.py)."""

from __future__ import annotations

import json
import os
from dataclasses import dataclass

import numpy as np

from oracle import mixing_ref

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load_json(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


@dataclass
class SamplingCase:
    name: str
    z: np.ndarray
    T: float
    top_k: int | None
    top_p: float
    u: np.ndarray
    tokens: np.ndarray
    kept: np.ndarray
    q: np.ndarray | None


def sampling_cases():
    d = np.load(os.path.join(GOLDEN, "sampling.npz"))
    out = []
    for i, name in enumerate(d["names"]):
        st, vocab, conc, bf = int(d["gen_state"][i]), int(d["gen_vocab"][i]), float(d["gen_conc"][i]), int(d["gen_bf16"][i])
        if bf < 0:
            z = d["rows"][d["rows_off"][i]: d["rows_off"][i + 1]].astype(np.float32)
        else:
            z = mixing_ref.fill_logits_np(st, vocab, conc, 5.0)
            if bf:
                z = mixing_ref.bf16_round(z)
        k = int(d["top_k"][i])
        qk = f"q_{i}"
        out.append(SamplingCase(
            str(name), z, float(d["T"][i]), None if k < 0 else k, float(d["top_p"][i]),
            d["u"][d["u_off"][i]: d["u_off"][i + 1]], d["tokens"][d["u_off"][i]: d["u_off"][i + 1]],
            d["kept"][d["kept_off"][i]: d["kept_off"][i + 1]], d[qk] if qk in d.files else None))
    return out
