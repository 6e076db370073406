#!/bin/bash
# balanced tile schedule (RAAS_SCHED=1) vs the unit-affine one: parity under mode 1, then A/B
RAAS_SCHED=1 timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
q() { python bench.py --no-e2e --no-cpu-baseline "$@" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('S=$RAAS_SCHED', '$*', round(d['roofline']['achieved']), 'GB/s', round(d['roofline']['avg_launch_us'],2), 'us', d['launch'], d['clocks']['sm_mhz'])"; }
for rep in 1 2; do
for s in 0 1; do
  export RAAS_SCHED=$s
  q --config 4 --steps 60 --warmup 5
  q --steps 100
  q --config 5 --L 256 --layers 8 --steps 100 --split-pages 8
  q --config 5 --L 256 --layers 8 --steps 100
  q --config 5 --L 512 --layers 8 --steps 100 --split-pages 16
  q --config 5 --L 1024 --layers 4 --steps 100
  q --config 2 --steps 200
done
done
