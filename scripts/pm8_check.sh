#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -3
bash scripts/ab.sh "--config 4 --steps 60;--steps 60;--config 5 --L 512 --layers 8 --steps 100" 2 build/ab_base.so build/ab_pm8.so 2>&1 | tee gpurun_out/pm8_ab.txt
RAAS_LIB=build/dbg.so timeout 300 python scripts/dbg_timing.py --B 32 --L 4096 --P 128 --Hq 28 --Hkv 4 --layers 8 2>&1 | tail -4
