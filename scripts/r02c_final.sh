#!/bin/bash
# GPU box, round-2 closing evidence on the final kernels (specialised instantiations): GPU test
# suite, smoke(), the headline bench 3x, every config / variant line, ncu launch lists + full
# captures of the config-3 decode kernel and of the specialised Quest-score kernel.
tag=${1:-r02c}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 2400 python -m pytest tests -m gpu -q --durations=8 > gpurun_out/pytest_${tag}.log 2>&1; tail -14 gpurun_out/pytest_${tag}.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for i in 1 2 3; do timeout 900 python bench.py 2>/dev/null | tee -a gpurun_out/bench3_${tag}.jsonl | cut -c1-150; done
bash scripts/run_configs.sh ${tag} > /dev/null 2>&1; wc -l gpurun_out/configs_${tag}.jsonl
prof() {  # name, skip, bench args...
  local name=$1 skip=$2; shift 2
  local ARGS="--steps 2 --warmup 3 --no-e2e --no-cpu-baseline $@"
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:raas_decode -s $skip -c 16 --csv --log-file gpurun_out/launches_${tag}_${name}.csv python bench.py $ARGS > /dev/null 2>&1; echo "$name list rc=$?"
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:raas_decode -s $skip -c 1 -o gpurun_out/prof_${tag}_${name} python bench.py $ARGS > gpurun_out/ncu_${tag}_${name}.log 2>&1; echo "$name full rc=$?"
}
prof cfg3 $((1900 * 32 + 1)) --fill 1900
prof cfg3_quest $((1900 * 32 + 1)) --fill 1900 --score quest
