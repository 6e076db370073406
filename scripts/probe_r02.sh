#!/bin/bash
# GPU box: consumer-time sensitivity probe at configs 4 and 3 (RAAS_DBG_DELAY / _HOLD builds)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
bash scripts/ab.sh "--config 4 --steps 60;--steps 60" 2 build/ab_base.so build/ab_nc.so build/ab_d300.so build/ab_d1000.so build/ab_h300.so build/ab_h1000.so 2>&1 | tee gpurun_out/probe_r02.txt
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 | tee gpurun_out/pytest_r02g.log
