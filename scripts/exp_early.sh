#!/bin/bash
python -m pytest tests -m gpu -q -x 2>&1 | tail -3
q() { python bench.py --no-e2e --no-cpu-baseline "$@" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$*', round(d['roofline']['achieved']), 'GB/s', round(d['roofline']['avg_launch_us'],2), 'us', d['ms_per_step'])"; }
for e in 0 1; do
  if [ $e = 1 ]; then export RAAS_NO_EARLY=1; fi
  echo "RAAS_NO_EARLY=$RAAS_NO_EARLY"
  q --steps 100
  q --config 2 --steps 200
  q --config 4 --steps 60
  q --config 5 --L 512 --layers 8 --steps 100
done
unset RAAS_NO_EARLY
RAAS_LIB=build_exp/libraas_dbg.so python scripts/timeline.py
RAAS_LIB=build_exp/libraas_dbg.so python scripts/timeline.py --B 1 --L 1024 --P 512 --sp 16 --layers 32
