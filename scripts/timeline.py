"""Tuning experiment: in-stream timeline of consecutive decode launches (RAAS_DBG_TIMING build,
RAAS_LIB=build_exp/libraas_dbg.so).  Config 3 shapes, `layers` distinct caches from a
full-cache state; prints per launch the spread of CTA entry, griddepcontrol.wait release,
producer end and exit (globaltimer, us, relative to the first launch's first release)."""
import ctypes, os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np, torch
from paper_2502_11147_b200 import raas
from paper_2502_11147_b200.raas import RaasLayer
from paper_2502_11147_b200.synth import random_steady_state
import argparse
ap = argparse.ArgumentParser()
ap.add_argument("--B", type=int, default=64); ap.add_argument("--L", type=int, default=2048)
ap.add_argument("--layers", type=int, default=8); ap.add_argument("--graph", type=int, default=1)
ap.add_argument("--P", type=int, default=256); ap.add_argument("--sp", type=int, default=0)
ap.add_argument("--Hq", type=int, default=32); ap.add_argument("--Hkv", type=int, default=8)
a = ap.parse_args()
B, Hq, Hkv, d, P, L = a.B, a.Hq, a.Hkv, 128, a.P, a.L
C, U = L // 16, B * Hkv
Pp = -(-P // 16)
meta = random_steady_state(77, U, C, Pp, Pp * 16 + 64 * (C - Pp) + 5)
layers = [RaasLayer(L, 1e-4, Hq, Hkv, d, B, split_pages=a.sp) for _ in range(a.layers)]
for ly in layers:
    ly.raas_set_state(meta["t"], meta["ts"], meta["start"], meta["count"], meta["pinned"])
q = torch.randn(B, Hq, d, device="cuda").bfloat16(); kv = torch.randn(B, Hkv, d, device="cuda").bfloat16()
out = torch.empty_like(q)
s = torch.cuda.Stream()
lib = raas.lib(); lib.raas_debug_timeline.argtypes = [ctypes.c_void_p, ctypes.c_int]
tl = np.zeros((8, 256, 4), np.uint64)
step = lambda: [ly.raas_decode_step(q, kv, kv, out, stream=s) for ly in layers]  # noqa: E731
with torch.cuda.stream(s):
    for _ in range(3):
        step()
torch.cuda.synchronize()
if a.graph:
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        step()
    with torch.cuda.stream(s):
        g.replay(); g.replay()
torch.cuda.synchronize()
lib.raas_debug_timeline(tl.ctypes.data_as(ctypes.c_void_p), tl.size)  # clear; slot counter reset
with torch.cuda.stream(s):
    for _ in range(max(1, 16 // a.layers)):
        g.replay() if a.graph else step()
torch.cuda.synchronize()
lib.raas_debug_timeline(tl.ctypes.data_as(ctypes.c_void_p), tl.size)
grid = layers[0].raas_launch_info()["grid"]
x = tl[:, :grid].astype(np.int64)
# launches were recorded into slots 0..7 in order, the last 8 kept: find the order by entry time
order = np.argsort(x[:, :, 1].min(1))
x = x[order]
t0 = x[0, :, 1].min()
r = (x - t0) / 1e3
nb = U * (4 * d * (L - 7.5) + 4 * d + 4 * (Hq // Hkv) * d + 12 * C)
print(f"grid {grid}; algorithmic bytes per launch {nb/1e6:.1f} MB")
print("launch | entry min/max | release min/max | prod end min/med/max | exit min/med/max | busy(us) | GB/s")
prev_exit = None
for k in range(8):
    e, w, pe, ex = r[k, :, 0], r[k, :, 1], r[k, :, 2], r[k, :, 3]
    busy = ex.max() - w.min()
    span = ex.max() - (prev_exit if prev_exit is not None else w.min())
    print(f"{k} | {e.min():7.1f} {e.max():7.1f} | {w.min():7.1f} {w.max():7.1f} | {pe.min():7.1f} {np.median(pe):7.1f} {pe.max():7.1f}"
          f" | {ex.min():7.1f} {np.median(ex):7.1f} {ex.max():7.1f} | {busy:6.1f} | {nb/span/1e3 if prev_exit is not None else 0:6.0f}")
    prev_exit = ex.max()
if os.environ.get("TL_DUMP"):
    np.save(os.environ["TL_DUMP"], r)  # [launch][cta][entry, release, producer end, exit] us
