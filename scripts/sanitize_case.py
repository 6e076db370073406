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
print("sanitize case ok", r1.max_err, r2.max_err, r3.max_err, r4.max_err, r5.max_err,
      r1.band_events + r2.band_events + r3.band_events + r4.band_events + r5.band_events)
