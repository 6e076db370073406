"""Tuning experiment: cycle accounting of the decode pipeline (needs a RAAS_DBG_TIMING build,
RAAS_LIB=build_exp/libraas_dbg.so).  Config 3 shapes, 1 layer, full-cache state."""
import ctypes, os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np, torch
from paper_2502_11147_b200 import raas
from paper_2502_11147_b200.raas import RaasLayer
from paper_2502_11147_b200.synth import random_steady_state
import argparse
ap = argparse.ArgumentParser()
ap.add_argument("--B", type=int, default=64); ap.add_argument("--Hq", type=int, default=32)
ap.add_argument("--Hkv", type=int, default=8); ap.add_argument("--L", type=int, default=2048)
ap.add_argument("--P", type=int, default=256); ap.add_argument("--sp", type=int, default=0)
ap.add_argument("--layers", type=int, default=8)
ap.add_argument("--table-scope", type=int, default=0)
ap.add_argument("--page", type=int, default=16)
ap.add_argument("--quest", type=int, default=0, help="Quest-on-prefill hybrid: prompt pages attended")
a = ap.parse_args()
B, Hq, Hkv, d, P, L = a.B, a.Hq, a.Hkv, 128, a.P, a.L
C, Pp, U = L // 16, P // 16, B * Hkv
Pp = -(-P // 16)
meta = random_steady_state(77, U, C, Pp, Pp * 16 + 64 * (C - Pp) + 5)
if a.table_scope:  # one table per request: replicate kv-head 0's state
    for k in ("t", "ts", "start", "count", "pinned"):
        v = meta[k].reshape(B, Hkv, *meta[k].shape[1:])
        meta[k] = np.ascontiguousarray(np.repeat(v[:, :1], Hkv, axis=1).reshape(meta[k].shape))
layers = [RaasLayer(L, 1e-4, Hq, Hkv, d, B, split_pages=a.sp, table_scope=a.table_scope, page=a.page,
                    quest_prefill_pages=a.quest)
          for _ in range(a.layers)]
print(layers[0].raas_launch_info())
q = torch.randn(B, Hq, d, device="cuda").bfloat16(); kv = torch.randn(B, Hkv, d, device="cuda").bfloat16()
out = torch.empty_like(q)
for ly in layers:
    if a.page == 16 and not a.quest:
        ly.raas_set_state(meta["t"], meta["ts"], meta["start"], meta["count"], meta["pinned"])
    else:  # token slots: prefill, then decode until every slot is used
        kp = torch.randn(B, Hkv, P, d, device="cuda").bfloat16()
        ly.raas_prefill(kp, kp, P)
        for i in range(L - P + 8 if a.page == 1 else (L - P) + 16):
            ly.raas_decode_step(q, kv, kv, out)
L_ = raas.lib(); L_.raas_debug_timing.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = np.zeros((1024, 16), np.uint64)
for i in range(4):
    for ly in layers: ly.raas_decode_step(q, kv, kv, out)
torch.cuda.synchronize()
L_.raas_debug_timing(buf.ctypes.data_as(ctypes.c_void_p), buf.size)
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
N = 16
for i in range(N):
    for ly in layers: ly.raas_decode_step(q, kv, kv, out)
e1.record(); torch.cuda.synchronize()
L_.raas_debug_timing(buf.ctypes.data_as(ctypes.c_void_p), buf.size)
ms = e0.elapsed_time(e1) / (N * len(layers))
g = layers[0].raas_launch_info()["grid"]
b = buf[:g].astype(np.float64).sum(0) / g / (N * len(layers))
names = {0: "prod tfree wait", 1: "prod empty wait (lane0)", 8: "prod total", 2: "merge mfull wait",
         7: "merge cq push wait", 9: "merge total", 4: "combine cq wait", 10: "combine total",
         5: "consumer full wait (sum 8 warps)", 6: "consumer q wait (sum)", 11: "consumer total (sum)"}
nbytes = U * (4 * d * (L - 7.5) + 4 * d + 4 * (Hq // Hkv) * d + 12 * C)
print(f"launch {ms*1e3:.1f} us  ({nbytes/(ms*1e-3)/1e9:.0f} GB/s)")
for k, n in names.items():
    print(f"{n:34s} {b[k]:12.0f} cyc/launch/CTA")

# one isolated launch: per-CTA start / producer end / combine end (globaltimer, ns)
torch.cuda.synchronize()
L_.raas_debug_timing(buf.ctypes.data_as(ctypes.c_void_p), buf.size)
layers[0].raas_decode_step(q, kv, kv, out)
torch.cuda.synchronize()
L_.raas_debug_timing(buf.ctypes.data_as(ctypes.c_void_p), buf.size)
st, pe, ce = buf[:g, 12].astype(np.int64), buf[:g, 13].astype(np.int64), buf[:g, 14].astype(np.int64)
t0 = st.min()
print("CTA start spread (us): min 0 max %.1f" % ((st.max() - t0) / 1e3))
print("producer end (us): min %.1f median %.1f max %.1f" % ((pe.min() - t0) / 1e3, np.median(pe - t0) / 1e3, (pe.max() - t0) / 1e3))
print("combine end  (us): min %.1f median %.1f max %.1f" % ((ce.min() - t0) / 1e3, np.median(ce - t0) / 1e3, (ce.max() - t0) / 1e3))
print("cycles/ns (SM clock GHz) ~ %.2f" % (buf[:g, 8].astype(np.float64).mean() / np.mean(pe - st)))

ub2 = np.zeros((4, 4096, 4), np.uint64)
L_.raas_debug_units.argtypes = [ctypes.c_void_p, ctypes.c_int]
L_.raas_debug_units(ub2.ctypes.data_as(ctypes.c_void_p), ub2.size)
ub = ub2[0, :U].astype(np.int64)
cm = ub2[1, :U].astype(np.int64)
push, cs, ce = (ub[:, 1] - t0) / 1e3, (ub[:, 2] - t0) / 1e3, (ub[:, 3] - t0) / 1e3
dur = ce - cs
order = np.argsort(-ce)[:6]
print("combine duration us: median %.1f max %.1f; queue delay median %.1f max %.1f" % (
    np.median(dur), dur.max(), np.median(cs - push), (cs - push).max()))
ph = (cm - ub[:, 2:3]) / 1e3  # combine phase marks relative to the combine start
print("combine phases (us from start, median): LSE %.2f  out %.2f  stamps %.2f  argmin %.2f  end %.2f" % (
    *np.median(ph, 0), np.median(dur)))
for u in order:
    print(f"  unit {u}: cta {ub[u,0]} pushed {push[u]:.1f} start {cs[u]:.1f} end {ce[u]:.1f}  phases {np.round(ph[u], 2)}")
cyc = ub2[2:].reshape(4096, 8)[:U].astype(np.int64)
print("fine marks recorded for", int((cyc[:, 6] != 0).sum()), "units")
if cyc[:, 6].any():
    d = np.diff(cyc[:, :7], axis=1)
    print("combine fine marks (SM cycles, median): (none) %d, load_meta %d, load_acc %d, a5 %d, "
          "stamp loop %d, argmin+plan %d" % tuple(np.median(d, 0)))
