#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
bash scripts/ab.sh "--config 4 --steps 60;--steps 60;--config 5 --L 512 --layers 8 --steps 100" 2 build/ab_pms.so build/ab_warm.so 2>&1 | tee gpurun_out/warm_ab.txt
for lib in dbg dbg_warm; do echo "== $lib"; RAAS_LIB=build/$lib.so timeout 300 python scripts/dbg_timing.py --B 32 --L 4096 --P 128 --Hq 28 --Hkv 4 --layers 8 2>&1 | tail -9; done
