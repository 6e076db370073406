#!/bin/bash
# GPU box: owned units' page maxima / metadata in shared memory (PmsCtx) -- parity + A/B
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "full_size_sampled or request_sharding or bitwise or toy or random_configs or interleaved or host_entry or graph" 2>&1 | tail -4
bash scripts/ab.sh "--config 4 --steps 60;--steps 60" 2 build/ab_base.so build/ab_pms.so 2>&1 | tee gpurun_out/pms_ab.txt
RAAS_LIB=build/dbg.so timeout 300 python scripts/dbg_timing.py --B 32 --L 4096 --P 128 --Hq 28 --Hkv 4 --layers 8 2>&1 | tail -12
