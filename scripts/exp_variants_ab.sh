#!/bin/bash
# A/B of two builds on the NEXT-row variants at config 3 shapes
q() { python bench.py --no-e2e --no-cpu-baseline --steps 60 "$@" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$*', round(d['roofline']['achieved']), 'GB/s', round(d['roofline']['avg_launch_us'],2), 'us', d['ms_per_step'])"; }
for f in "$@"; do
  echo "== $f"
  for v in "--score quest" "--top-r 0.5" "--table-scope 1" "--page 1"; do RAAS_LIB=$f q $v; done
done
