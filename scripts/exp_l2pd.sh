#!/bin/bash
# L2 prefetch distance ahead of the ring (RAAS_L2PD builds)
q() { RAAS_LIB=$1 python bench.py --no-e2e --no-cpu-baseline "${@:2}" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$(basename $1 .so)', '${*:2}', round(d['roofline']['achieved']), 'GB/s', round(d['roofline']['avg_launch_us'],2), 'us', d['clocks']['sm_mhz'])"; }
for rep in 1 2; do for f in "$@"; do
  q $f --steps 100
  q $f --config 4 --steps 60
  q $f --config 2 --steps 200
  q $f --config 5 --L 512 --layers 8 --steps 100
  q $f --config 5 --L 4096 --layers 4 --steps 60
done; done
