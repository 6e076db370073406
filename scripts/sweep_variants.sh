#!/bin/bash
# GPU box: bench each build_exp/libraas_*.so (tuning experiments) on config 3, short runs.
mkdir -p gpurun_out
for f in ${@:-build_exp/libraas_*.so}; do
  n=$(basename $f .so)
  r=$(RAAS_LIB=$f python bench.py --steps 100 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(f\"{d['roofline']['achieved']:.0f} GB/s  {d['ms_per_step']:.3f} ms/step  launch={d['launch']}\")")
  echo "$n: $r"
done
