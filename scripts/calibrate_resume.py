"""Calibrate the waterfall query strength lambda of synth.waterfall_resume per full-size config so
that the oracle's page stamp rate lands in the 30-60 % band of SURVEY §8(d) (test input recipe,
DESIGN.md §4).  Runs the CPU oracle only, on the sampled requests (first and last)."""
import sys
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
from paper_2502_11147_b200.synth import waterfall_resume  # noqa: E402

CFGS = {2: (1, 32, 8, 1024, 512), 3: (64, 32, 8, 2048, 256), 4: (32, 28, 4, 4096, 128),
        "5a": (8, 32, 8, 8192, 128), "5b": (16, 32, 8, 256, 128)}


def rate(cfg, lam, T=48, cur=5, seed=81):
    B, Hq, Hkv, L, P = cfg
    Bs = 2 if B > 1 else 1
    st, ks, vs, steps = waterfall_resume(seed, Bs, Hq, Hkv, 128, L, P, T, cur_count=cur, lam=lam)
    o = oracle.Oracle(L=L, alpha=1e-4, page=16, n_q_heads=Hq, n_kv_heads=Hkv, head_dim=128, batch=Bs)
    o.set_state(st["t"], st["ts"], st["start"], st["count"], st["pinned"], ks, vs)
    dec = stamp = ev = 0
    for i in range(T):
        o.decode_step(steps.q[i], steps.k[i], steps.v[i], want_out=False)
        tr = o.get_trace()
        ps = tr["pstar"]
        dec += int((ps >= 0).sum())
        stamp += int((ps > 1e-4).sum())
        ev += int((tr["evicted"] >= 0).sum())
    return stamp / dec, ev


if __name__ == "__main__":
    oracle.set_threads(0)
    keys = sys.argv[1:] or list(CFGS)
    for k in keys:
        k = int(k) if k.isdigit() else k
        for lam in [float(x) for x in os.environ.get("LAMS", "4,5,6,7,8").split(",")]:
            r, ev = rate(CFGS[k], lam)
            print(f"config {k} lambda {lam}: stamp rate {r:.3f}, evictions {ev}", flush=True)
