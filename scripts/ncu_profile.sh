#!/bin/bash
# GPU box: ncu launch list + one full capture of the decode kernel at steady state (config 3).
tag=${1:-dev}; shift
mkdir -p gpurun_out
ARGS="--fill 1900 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline $@"
SKIP=60850
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:raas_decode -s $SKIP -c 64 --csv --log-file gpurun_out/launches_${tag}.csv python bench.py $ARGS > /dev/null 2>&1; echo "ncu list rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:raas_decode -s $SKIP -c 1 -o gpurun_out/prof_${tag} python bench.py $ARGS > gpurun_out/ncu_${tag}.log 2>&1; echo "ncu full rc=$?"; tail -2 gpurun_out/ncu_${tag}.log
