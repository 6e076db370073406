"""Small lockstep case for compute-sanitizer runs (memcheck / racecheck / synccheck / initcheck):
toy config plus a multi-tile Llama-shaped case, GPU vs oracle."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import oracle
from lockstep import run_lockstep
from paper_2502_11147_b200.synth import waterfall_stream
st = waterfall_stream(1000, 1, 4, 2, 64, 32, 40)
r1, _, _ = run_lockstep(oracle, st, L=64, alpha=1e-4, Hq=4, Hkv=2)
st = waterfall_stream(7, 2, 8, 2, 128, 40, 30)
r2, _, _ = run_lockstep(oracle, st, L=256, alpha=1e-4, Hq=8, Hkv=2, split_pages=4)
st = waterfall_stream(8, 2, 8, 2, 128, 40, 30)
r3, _, _ = run_lockstep(oracle, st, L=256, alpha=1e-4, Hq=8, Hkv=2, split_pages=4, table_scope=1)
st = waterfall_stream(9, 2, 8, 2, 128, 37, 60)
r4, _, _ = run_lockstep(oracle, st, L=96, alpha=1e-3, Hq=8, Hkv=2, split_pages=2, page=1, state_every=4)
r5, _, _ = run_lockstep(oracle, st, L=96, alpha=1e-3, Hq=8, Hkv=2, split_pages=2, page=1, table_scope=1)
# cluster schedule (B = 1: each unit's 4 split CTAs exchange partials through distributed
# shared memory), from the prompt on, so the fill phase's empty splits are exercised
st = waterfall_stream(10, 1, 32, 8, 128, 100, 90)
r6, ly6, _ = run_lockstep(oracle, st, L=512, alpha=1e-4, Hq=32, Hkv=8, split_pages=8)
assert ly6.raas_launch_info()["cluster"] == 4
print("sanitize case ok", r1.max_err, r2.max_err, r3.max_err, r4.max_err, r5.max_err, r6.max_err,
      r1.band_events + r2.band_events + r3.band_events + r4.band_events + r5.band_events + r6.band_events)

# early start (two handles interleaved on one stream) and the zero-copy host path
import numpy as np, torch
from paper_2502_11147_b200.raas import RaasLayer


def bits_dev(x):
    return torch.from_numpy(np.ascontiguousarray(x).view(np.int16)).view(torch.bfloat16).cuda()


sts = [waterfall_stream(20 + i, 2, 8, 2, 128, 40, 24) for i in range(2)]
lys = []
for st in sts:
    ly = RaasLayer(96, 1e-4, 8, 2, 128, 2)
    ly.raas_prefill(bits_dev(st.k_pre), bits_dev(st.v_pre), 40)
    lys.append(ly)
out = torch.empty((2, 8, 128), dtype=torch.bfloat16, device="cuda")
for i in range(24):
    for st, ly in zip(sts, lys):
        ly.raas_decode_step(bits_dev(st.q[i]), bits_dev(st.k[i]), bits_dev(st.v[i]), out)
pin = lambda x: torch.from_numpy(np.ascontiguousarray(x).view(np.int16)).view(torch.bfloat16).pin_memory()  # noqa: E731
oh = torch.empty((2, 8, 128), dtype=torch.bfloat16).pin_memory()
st = waterfall_stream(30, 2, 8, 2, 128, 40, 8)
for i in range(8):
    lys[0].raas_decode_step_host(pin(st.q[i]), pin(st.k[i]), pin(st.v[i]), oh)
torch.cuda.synchronize()
assert all(ly.raas_get_status() == 0 for ly in lys)
print("sanitize early/host ok")
