#!/bin/bash
# Config 2 (B = 1, L = 1024): split-size x grid sweep (us per launch)
q() { python bench.py --config 2 --no-e2e --no-cpu-baseline --steps 200 "$@" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$*', 'G=%s' % d['launch']['grid'], 'SP=%s' % d['launch']['split_pages'], round(d['roofline']['avg_launch_us'],2), 'us')"; }
for sp in 2 4 8 16 32; do
  q --split-pages $sp
  for G in 16 32 64 128 148; do RAAS_GRID=$G q --split-pages $sp; done
done
