"""Input builders for the hand-traced pins (P3, P3') — shared by CPU and GPU tests.

These only construct q/k/v from the golden files' recipes (tests/golden/*.json); the
expected results live in the golden files and were derived by hand from PAPER.md.
"""
import json
import os

import numpy as np

from paper_2502_11147_b200.synth import Stream, bf16_bits

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load_golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def hand_trace_stream():
    """P3: token level, P=2, L=6, d=16.  Returns (golden, Stream)."""
    g = load_golden("p3_hand_trace.json")
    s = g["setup"]
    d, P = s["head_dim"], s["P"]
    S = {int(k): set(v) for k, v in s["stamp_sets"].items()}
    E = np.eye(d, dtype=np.float32)
    T = 12 - P
    k_pre = np.stack([E[j - 1] for j in range(1, P + 1)])[None, None]
    q = np.zeros((T, 1, 1, d), np.float32)
    k = np.zeros((T, 1, 1, d), np.float32)
    for i, t in enumerate(range(P + 1, 13)):
        q[i, 0, 0] = 48.0 * sum(E[j - 1] for j in (S.get(t, set()) | {t}))
        k[i, 0, 0] = E[t - 1]
    zeros_pre = np.zeros((1, 1, P, d), np.float32)
    zeros = np.zeros((T, 1, 1, d), np.float32)
    return g, Stream(bf16_bits(k_pre), bf16_bits(zeros_pre), bf16_bits(q), bf16_bits(k), bf16_bits(zeros))


def page_twin_stream(g_heads=1, value_seed=None):
    """P3': page 16, P=32, L=96, d=64.  Optionally replicate the query over a GQA group
    and give the tokens random values (the values do not affect the bookkeeping)."""
    g = load_golden("p3_page_twin.json")
    s = g["setup"]
    d, P, T = s["head_dim"], s["P"], s["decode_steps"]
    S = {int(k): set(v) for k, v in s["stamp_sets"].items()}
    E = np.eye(d, dtype=np.float32)
    page = s["page"]
    k_pre = np.stack([E[j // page + 1] for j in range(P)])[None, None]
    q = np.zeros((T, 1, g_heads, d), np.float32)
    k = np.zeros((T, 1, 1, d), np.float32)
    for i, t in enumerate(range(P + 1, P + T + 1)):
        e = (t - 1) // page + 1
        q[i, 0, :] = 96.0 * sum(E[m] for m in (S.get(e, set()) | {e}))
        k[i, 0, 0] = E[e]
    if value_seed is None:
        v_pre = np.zeros((1, 1, P, d), np.float32)
        v = np.zeros((T, 1, 1, d), np.float32)
    else:
        rng = np.random.default_rng(value_seed)
        v_pre = rng.standard_normal((1, 1, P, d)).astype(np.float32)
        v = rng.standard_normal((T, 1, 1, d)).astype(np.float32)
    return g, Stream(bf16_bits(k_pre), bf16_bits(v_pre), bf16_bits(q), bf16_bits(k), bf16_bits(v))
