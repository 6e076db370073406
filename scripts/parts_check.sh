#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -3
bash scripts/ab.sh "--config 4 --steps 60;--steps 60;--config 5 --L 512 --layers 8 --steps 100;--config 5 --L 1024 --layers 8 --steps 100" 2 build/ab_base.so build/ab_parts.so 2>&1 | tee gpurun_out/parts_ab.txt
for lib in ab_base ab_parts; do RAAS_LIB=build/$lib.so timeout 600 python bench.py --no-cpu-baseline --steps 100 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib e2e', round(d['e2e']['value'],1), 'dev', round(d['value'],1))"; done | tee -a gpurun_out/parts_ab.txt
