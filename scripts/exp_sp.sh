#!/bin/bash
q() { python bench.py --no-e2e --no-cpu-baseline "$@" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$*', round(d['roofline']['achieved']), 'GB/s', round(d['roofline']['avg_launch_us'],2), 'us', d['launch']['grid'], d['launch']['split_pages'])"; }
for f in paper_2502_11147_b200/libraas.so build_exp/libraas_outpipe.so; do
  echo "== $f"
  for sp in 32 64; do
    RAAS_LIB=$f q --config 4 --steps 60 --split-pages $sp
    RAAS_LIB=$f q --config 5 --L 8192 --layers 4 --steps 60 --split-pages $sp
  done
  RAAS_LIB=$f q --steps 100
  RAAS_LIB=$f q --steps 100 --split-pages 64
done
