#!/bin/bash
# GPU box: waterfall-data bench + L2-prefetch depth experiment (in-stream and isolated).
mkdir -p gpurun_out
python bench.py 2> gpurun_out/bench_wf_stderr.log > gpurun_out/bench_wf.json; cut -c1-300 gpurun_out/bench_wf.json; tail -2 gpurun_out/bench_wf_stderr.log
python bench.py --data gaussian --steps 100 --no-e2e --no-cpu-baseline 2>/dev/null | cut -c1-200
bash scripts/sweep_variants.sh build_exp/libraas_pf0.so build_exp/libraas_pf1.so build_exp/libraas_pf3.so paper_2502_11147_b200/libraas.so
for f in build_exp/libraas_pf0.so paper_2502_11147_b200/libraas.so; do
  n=$(basename $f .so)
  RAAS_LIB=$f timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:raas_decode -s 60850 -c 32 --csv --log-file gpurun_out/launches_$n.csv python bench.py --fill 1900 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo "ncu $n rc=$?"
done
