"""Tuning experiment: per-step time of the hybrid (Quest-on-prefill) mode vs plain, eager and
graph, config-3 shapes with a 1024-token prompt."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np, torch
from paper_2502_11147_b200.raas import RaasLayer
from paper_2502_11147_b200.synth import random_steady_state
B, Hq, Hkv, d, P, L = 64, 32, 8, 128, 1024, 2048
C, Pp, U = L // 16, P // 16, B * Hkv
meta = random_steady_state(77, U, C, Pp, Pp * 16 + 64 * (C - Pp) + 5)
rng = np.random.default_rng(0)
for K in (0, 16):
    layers = [RaasLayer(L, 1e-4, Hq, Hkv, d, B, quest_prefill_pages=K) for _ in range(4)]
    for ly in layers:
        ly.raas_set_state(meta["t"], meta["ts"], meta["start"], meta["count"], meta["pinned"])
    q = torch.randn(B, Hq, d, device="cuda").bfloat16(); kv = torch.randn(B, Hkv, d, device="cuda").bfloat16()
    out = torch.empty_like(q)
    for _ in range(3):
        for ly in layers: ly.raas_decode_step(q, kv, kv, out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(20):
        for ly in layers: ly.raas_decode_step(q, kv, kv, out)
    e1.record(); torch.cuda.synchronize()
    print(f"K={K}: eager {e0.elapsed_time(e1) / 80 * 1e3:.1f} us per layer-step")
