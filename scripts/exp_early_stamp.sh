#!/bin/bash
# A/B: first metadata chunk stamped before the output fold (libraas.so) vs before (libraas_base.so)
q() { RAAS_LIB=$1 python bench.py --no-e2e --no-cpu-baseline "${@:2}" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$(basename $1 .so)', '${*:2}', round(d['roofline']['achieved']), 'GB/s', round(d['roofline']['avg_launch_us'],2), 'us', d['clocks']['sm_mhz'])"; }
e() { RAAS_LIB=$1 python bench.py --no-cpu-baseline --steps 100 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$(basename $1 .so)', 'e2e cfg3', 'device', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), d['clocks']['sm_mhz'])"; }
for rep in 1 2; do
  for f in build_exp/libraas_base.so paper_2502_11147_b200/libraas.so; do
    q $f --config 2 --steps 200
    q $f --steps 100
    q $f --config 4 --steps 60
    q $f --config 5 --L 256 --layers 8 --steps 100
    q $f --config 5 --L 4096 --layers 4 --steps 60
    q $f --config 5 --L 8192 --layers 4 --steps 40
    e $f
  done
done
