#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -k "quest or variants or interleaved or set_state or host_entry" 2>&1 | tail -3
bash scripts/ab.sh "--steps 60 --score quest;--config 4 --steps 60 --score quest" 2 build/ab_base.so build/ab_qst.so 2>&1 | tee gpurun_out/qst_ab.txt
