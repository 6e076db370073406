"""Repro helper: full-cache state (random_steady_state), a few decode steps, B and L from argv."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np, torch
from paper_2502_11147_b200.raas import RaasLayer
from paper_2502_11147_b200.synth import bf16_bits, random_steady_state
B = int(sys.argv[1]) if len(sys.argv) > 1 else 1
L = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
sp = int(sys.argv[3]) if len(sys.argv) > 3 else 0
Hq, Hkv, d, P = 32, 8, 128, 256
C, Pp, U = L // 16, P // 16, B * Hkv
meta = random_steady_state(77, U, C, Pp, Pp * 16 + 64 * (C - Pp) + 5)
rng = np.random.Generator(np.random.Philox(78))
ks = bf16_bits(rng.standard_normal((U, C, 16, d), np.float32))
layer = RaasLayer(L, 1e-4, Hq, Hkv, d, B, split_pages=sp)
print(layer.raas_launch_info(), flush=True)
layer.raas_set_state(meta["t"], meta["ts"], meta["start"], meta["count"], meta["pinned"], ks, ks)
q = torch.randn(B, Hq, d, device="cuda").bfloat16()
kv = torch.randn(B, Hkv, d, device="cuda").bfloat16()
out = torch.empty_like(q)
for i in range(3):
    layer.raas_decode_step(q, kv, kv, out)
    torch.cuda.synchronize()
    print("step", i, "ok", layer.raas_get_status(), flush=True)
