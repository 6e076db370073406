"""Repro helper: lockstep at L=2048 with 32-page splits on a small batch."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import oracle
from lockstep import run_lockstep
from paper_2502_11147_b200.synth import waterfall_stream
sp = int(sys.argv[1]) if len(sys.argv) > 1 else 32
st = waterfall_stream(5, 1, 8, 2, 128, 64, int(sys.argv[2]) if len(sys.argv) > 2 else 40)
res, layer, _ = run_lockstep(oracle, st, L=2048, alpha=1e-4, Hq=8, Hkv=2, split_pages=sp)
print("ok", sp, res.max_err, res.band_events)
