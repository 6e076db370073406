#!/bin/bash
# per-SM streaming ceiling + in-stream timelines at config 4 and the small-L sweep point
./scripts/bw_probe
export RAAS_LIB=build_exp/libraas_dbg.so
python scripts/timeline.py --B 32 --Hq 28 --Hkv 4 --L 4096 --P 128
RAAS_GRID=148 python scripts/timeline.py --B 32 --Hq 28 --Hkv 4 --L 4096 --P 128
python scripts/timeline.py --B 64 --L 256 --P 128
RAAS_GRID=148 python scripts/timeline.py --B 64 --L 256 --P 128
