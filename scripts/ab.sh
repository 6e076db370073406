#!/bin/bash
# GPU box: interleaved A/B of alternative builds of libraas (tuning experiments).
#   scripts/ab.sh "<bench args>;<bench args>;..." <reps> lib1.so lib2.so ...
# Each case is a bench.py argument string; every (rep, lib, case) prints one line:
#   <lib> | <case> | GB/s | us per launch | SM MHz
cases=$1; reps=$2; shift 2
q() { RAAS_LIB=$1 timeout 600 python bench.py --no-e2e --no-cpu-baseline $2 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$(basename $1 .so) | $2 |', round(d['roofline']['achieved']), 'GB/s |', round(d['roofline']['avg_launch_us'],2), 'us |', d['clocks']['sm_mhz'], 'MHz')" || echo "$(basename $1 .so) | $2 | FAILED"; }
IFS=';' read -ra CS <<< "$cases"
for rep in $(seq 1 $reps); do
  for f in "$@"; do
    for c in "${CS[@]}"; do q $f "$c"; done
  done
done
