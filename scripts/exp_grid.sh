#!/bin/bash
# grid / split-size sweep at the configs whose unit count does not fill 148 SMs evenly
q() { python bench.py --no-e2e --no-cpu-baseline "$@" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$RAAS_GRID', '$*', round(d['roofline']['achieved']), 'GB/s', round(d['roofline']['avg_launch_us'],2), 'us', d['launch'], d['clocks']['sm_mhz'])"; }
for G in 0 148; do for sp in 0 16; do RAAS_GRID=$G q --config 4 --steps 60 --warmup 5 --split-pages $sp; done; done
for G in 0 148; do for sp in 0 8; do RAAS_GRID=$G q --config 5 --L 256 --layers 8 --steps 100 --split-pages $sp; done; done
for G in 0 148; do for sp in 0 16; do RAAS_GRID=$G q --config 5 --L 512 --layers 8 --steps 100 --split-pages $sp; done; done
