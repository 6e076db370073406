#!/bin/bash
# grid override at the configs where the chooser mixes owned and shared units
q() { python bench.py --no-e2e --no-cpu-baseline "$@" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('G=$RAAS_GRID', '$*', round(d['roofline']['achieved']), 'GB/s', round(d['roofline']['avg_launch_us'],2), 'us', d['launch']['grid'], d['clocks']['sm_mhz'])"; }
for rep in 1 2; do for G in 0 128 137 146; do
  export RAAS_GRID=$G
  q --steps 100
  q --config 5 --L 1024 --layers 4 --steps 100
  q --config 5 --L 4096 --layers 4 --steps 60
done; done
