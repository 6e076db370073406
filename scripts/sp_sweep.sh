#!/bin/bash
# GPU box: split-size / config sweep (tuning): prints GB/s and us per launch
q() { python bench.py --no-e2e --no-cpu-baseline "$@" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$*', round(d['roofline']['achieved']), 'GB/s', round(d['roofline']['avg_launch_us'],1), 'us', d['launch'])"; }
q --config 3 --steps 200
q --config 4 --steps 100
for sp in 2 4 8 16; do q --config 2 --steps 200 --split-pages $sp; done
for sp in 4 8 16; do q --config 5 --L 256 --layers 8 --steps 100 --split-pages $sp; done
for sp in 8 16 32; do q --config 5 --L 512 --layers 8 --steps 100 --split-pages $sp; done
for sp in 16 32; do q --config 5 --L 1024 --layers 4 --steps 100 --split-pages $sp; done
