#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -k "quest or variants or interleaved or set_state or host_entry or top_r or request_table or hybrid or checked" 2>&1 | tail -3
bash scripts/ab.sh "--steps 60 --score quest;--steps 60 --top-r 0.5;--steps 60 --table-scope 1;--steps 60 --P 1024 --quest-prefill 16" 2 build/ab_base.so build/ab_fm.so 2>&1 | tee gpurun_out/fm_ab.txt
