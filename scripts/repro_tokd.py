"""Debug: deferred token-level stamping (tokd) vs the oracle on config variants; prints every
mismatching row at the first failing readout."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np, torch
import oracle
from lockstep import to_dev
from paper_2502_11147_b200.raas import RaasLayer
from paper_2502_11147_b200.synth import waterfall_stream
cases = [  # B, Hq, Hkv, d, P, T, L, sp, every




    (2, 28, 4, 128, 37, 260, 192, 3, 2),
]
for c in cases:
    B, Hq, Hkv, d, P, T, L, sp, every = c
    st = waterfall_stream(700 + B + Hq + P, B, Hq, Hkv, d, P, T)
    ly = RaasLayer(L, 1e-3, Hq, Hkv, d, B, split_pages=sp, page=1)
    ly.raas_prefill(to_dev(st.k_pre), to_dev(st.v_pre), P)
    o = oracle.Oracle(L=L, alpha=1e-3, page=1, n_q_heads=Hq, n_kv_heads=Hkv, head_dim=d, batch=B)
    o.prefill(st.k_pre, st.v_pre, P)
    out = torch.empty((B, Hq, d), dtype=torch.bfloat16, device="cuda")
    hist = []
    bad = None
    for i in range(T):
        ly.raas_decode_step(to_dev(st.q[i]), to_dev(st.k[i]), to_dev(st.v[i]), out)
        o.decode_step(st.q[i], st.k[i], st.v[i], want_out=False)
        hist.append(o.get_trace()["pstar"].copy())
        if (i + 1) % every == 0:
            g, ob = ly.raas_get_state(), o.get_state()
            if not np.array_equal(g["ts"], ob["ts"]) or not np.array_equal(g["start"], ob["start"]):
                diff = np.argwhere(g["ts"] != ob["ts"])
                t = int(ob["t"][0])
                print(c, f"step t={t} used={int((g['count'][0] > 0).sum())} start_eq={np.array_equal(g['start'], ob['start'])}")
                for u, p in diff[:8]:
                    gt, ot = int(g["ts"][u, p]), int(ob["ts"][u, p])
                    tau = max(gt, ot)
                    ps = hist[-1 - (t - tau)][u, p] if 0 <= t - tau < len(hist) else -9
                    print(f"   unit {u} slot {p} (tile {p // 16} row {p % 16}) gpu ts {gt} oracle {ot} start {int(ob['start'][u, p])} p*@{tau}={ps:.3g}")
                bad = True
                break
            hist = []
    if not bad:
        print(c, "ok")
    print("status", ly.raas_get_status())
    if os.environ.get("RAAS_LIB", "").endswith("tokdbg.so"):
        import ctypes
        from paper_2502_11147_b200 import raas as R
        buf = np.zeros(16, np.int32)
        R.lib().raas_debug_tokd(buf.ctypes.data_as(ctypes.c_void_p))
        print("dbg unit,page,k,par,tm1,pend,smem,glob,cta,w,r,ks,flags:", buf[:13].tolist())
        print("launch", ly.raas_launch_info())
