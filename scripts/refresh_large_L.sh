#!/bin/bash
# GPU box: refresh the configs table and the L = 8192 ncu evidence after a kernel change that
# only the large budgets see (prefetch depth cap)
tag=${1:-r01}
bash scripts/run_configs.sh ${tag} > /dev/null
mkdir -p gpurun_out
ARGS="--steps 2 --warmup 3 --no-e2e --no-cpu-baseline --config 5 --L 8192 --layers 4 --fill 8100"
skip=$((8100 * 4 + 1))
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:raas_decode -s $skip -c 16 --csv --log-file gpurun_out/launches_${tag}_cfg5_L8192.csv python bench.py $ARGS > /dev/null 2>&1; echo "list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:raas_decode -s $skip -c 1 -o gpurun_out/prof_${tag}_cfg5_L8192 python bench.py $ARGS > gpurun_out/ncu_${tag}_cfg5_L8192.log 2>&1; echo "full rc=$?"
