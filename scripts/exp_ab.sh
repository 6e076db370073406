#!/bin/bash
# A/B of two builds (RAAS_LIB) on configs 3 / 2 / 4, alternating to average out drift
q() { python bench.py --no-e2e --no-cpu-baseline "$@" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$*', round(d['roofline']['achieved']), 'GB/s', round(d['roofline']['avg_launch_us'],2), 'us')"; }
for rep in 1 2; do
for f in "$@"; do
  echo "== $f"
  RAAS_LIB=$f q --steps 100
  RAAS_LIB=$f q --config 2 --steps 200
  RAAS_LIB=$f q --config 4 --steps 60
done
done
