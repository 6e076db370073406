"""Full-size steps for the checked build (-DRAAS_CHECKED: device bounds checks reported in the
status word): configs 2-5 shapes from full-cache waterfall states, and the method variants at
config 3 shapes.  Run with RAAS_LIB pointing at the checked library; prints one line per case."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2502_11147_b200.raas import RaasLayer  # noqa: E402
from paper_2502_11147_b200.synth import waterfall_resume  # noqa: E402


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x).view(np.int16)).view(torch.bfloat16).cuda()


cases = [  # B, Hq, Hkv, L, P, split_pages, options
    (64, 32, 8, 2048, 256, 0, {}),                                  # config 3
    (32, 28, 4, 4096, 128, 0, {}),                                  # config 4 (per GPU)
    (1, 32, 8, 1024, 512, 16, {}),                                  # config 2 (cluster schedule)
    (16, 32, 8, 256, 128, 0, {}),                                   # config 5, L = 256 (half CTAs)
    (8, 32, 8, 8192, 128, 0, {}),                                   # config 5, L = 8192
    (16, 32, 8, 2048, 256, 0, {"score_mode": 1}),                   # Quest scores
    (16, 32, 8, 2048, 256, 0, {"stamp_rule": 1, "top_r": 0.5}),     # top-r
    (16, 32, 8, 2048, 256, 0, {"table_scope": 1}),                  # one table per request
]
for B, Hq, Hkv, L, P, sp, kw in cases:
    d, T = 128, 24
    st, kst, vst, steps = waterfall_resume(5 + L + B, B, Hq, Hkv, d, L, P, T, cur_count=7, lam=7.0)
    if kw.get("table_scope"):  # one state replica per request: copy kv-head 0's
        for k in ("t", "ts", "start", "count", "pinned"):
            v = st[k].reshape(B, Hkv, *st[k].shape[1:])
            st[k] = np.ascontiguousarray(np.repeat(v[:, :1], Hkv, axis=1).reshape(st[k].shape))
        for a in (kst, vst):
            v = a.reshape(B, Hkv, *a.shape[1:])
            a[:] = np.repeat(v[:, :1], Hkv, axis=1).reshape(a.shape)
    layer = RaasLayer(L, 1e-4, Hq, Hkv, d, B, split_pages=sp, **kw)
    layer.raas_set_state(st["t"], st["ts"], st["start"], st["count"], st["pinned"], kst, vst)
    out = torch.empty((B, Hq, d), dtype=torch.bfloat16, device="cuda")
    for i in range(T):
        layer.raas_decode_step(dev(steps.q[i]), dev(steps.k[i]), dev(steps.v[i]), out)
    status = layer.raas_get_status()
    print(f"checked case B={B} L={L} sp={sp} {kw} {layer.raas_launch_info()}: status {status:#x}")
    assert status == 0, hex(status)
print("checked cases ok")
