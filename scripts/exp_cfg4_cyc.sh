#!/bin/bash
# cycle accounting at config 4 vs config 3 shapes; pipeline ceiling without compute
for lib in build_exp/libraas_dbg.so build_exp/libraas_nocomp.so; do
  echo "== $lib"
  RAAS_LIB=$lib python scripts/dbg_timing.py --B 32 --Hq 28 --Hkv 4 --L 4096 --P 128 2>&1 | head -20
  RAAS_LIB=$lib python scripts/dbg_timing.py 2>&1 | head -20
done
