#!/bin/bash
# GPU box: ncu launch list + one full capture of the decode kernel at steady state for the other
# config 4 (G=1, 32 requests, L=4096) and config 5 at L=256 / L=8192.
tag=${1:-dev}
mkdir -p gpurun_out
prof() {  # name, skip, bench args...
  local name=$1 skip=$2; shift 2
  local ARGS="--steps 2 --warmup 3 --no-e2e --no-cpu-baseline $@"
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:raas_decode -s $skip -c 16 --csv --log-file gpurun_out/launches_${tag}_${name}.csv python bench.py $ARGS > /dev/null 2>&1; echo "$name list rc=$?"
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:raas_decode -s $skip -c 1 -o gpurun_out/prof_${tag}_${name} python bench.py $ARGS > gpurun_out/ncu_${tag}_${name}.log 2>&1; echo "$name full rc=$?"
}
prof cfg4 $((4000 * 28 + 1)) --config 4 --fill 4000
prof cfg5_L256 $((200 * 8 + 1)) --config 5 --L 256 --layers 8 --fill 200
prof cfg5_L8192 $((8100 * 4 + 1)) --config 5 --L 8192 --layers 4 --fill 8100
