#!/bin/bash
# GPU box, round-2 evidence part B: ncu launch list (16 steady-state launches) + one --set full
# capture of the decode kernel per config (commands per B200_PROFILING.md; 1 GPU).
tag=${1:-r02}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
prof() {  # name, skip, bench args...
  local name=$1 skip=$2; shift 2
  local ARGS="--steps 2 --warmup 3 --no-e2e --no-cpu-baseline $@"
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:raas_decode -s $skip -c 16 --csv --log-file gpurun_out/launches_${tag}_${name}.csv python bench.py $ARGS > /dev/null 2>&1; echo "$name list rc=$?"
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:raas_decode -s $skip -c 1 -o gpurun_out/prof_${tag}_${name} python bench.py $ARGS > gpurun_out/ncu_${tag}_${name}.log 2>&1; echo "$name full rc=$?"
}
prof cfg3 $((1900 * 32 + 1)) --fill 1900
# same launches with L2 left warm between kernels (ncu flushes caches by default)
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:raas_decode -s $((1900 * 32 + 1)) -c 16 --csv --log-file gpurun_out/launches_${tag}_cfg3_warm.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --fill 1900 > /dev/null 2>&1; echo "cfg3 warm list rc=$?"
prof cfg4 $((4000 * 28 + 1)) --config 4 --fill 4000
prof cfg2 $((600 * 4 * 32 + 1)) --config 2 --fill 600
prof cfg5_L256 $((200 * 8 + 1)) --config 5 --L 256 --layers 8 --fill 200
prof cfg3_quest $((1900 * 32 + 1)) --fill 1900 --score quest
