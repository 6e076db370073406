#!/bin/bash
q() { python bench.py --no-e2e --no-cpu-baseline "$@" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$*', round(d['roofline']['achieved']), 'GB/s', round(d['roofline']['avg_launch_us'],1), 'us', d['launch'])"; }
for G in 0 148 144 136; do RAAS_GRID=$G q --config 4 --steps 60 --warmup 5; done
for G in 0 148; do RAAS_GRID=$G q --config 5 --L 1024 --layers 4 --steps 100; done
for G in 0 148; do RAAS_GRID=$G q --config 5 --L 512 --layers 8 --steps 100; done
