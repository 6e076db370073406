#!/bin/bash
# GPU box, round-2 final evidence: the GPU test suite, smoke(), the headline line, every config,
# kernel traces (configs 3, 4, 2, hybrid) and ncu of the cluster-schedule kernel (config 2).
tag=${1:-r02f}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 2400 python -m pytest tests -m gpu -q --durations=8 > gpurun_out/pytest_${tag}.log 2>&1; tail -12 gpurun_out/pytest_${tag}.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py 2> gpurun_out/bench_${tag}_stderr.log > gpurun_out/bench_${tag}.json; cut -c1-200 gpurun_out/bench_${tag}.json
for c in 3 4 2; do timeout 600 python bench.py --config $c --steps 20 --no-e2e --no-cpu-baseline --trace gpurun_out/trace_${tag}_cfg$c.json > /dev/null 2>&1; done
timeout 600 python bench.py --steps 20 --no-e2e --no-cpu-baseline --P 1024 --quest-prefill 16 --trace gpurun_out/trace_${tag}_hybrid.json > /dev/null 2>&1
bash scripts/run_configs.sh ${tag} > /dev/null 2>&1; wc -l gpurun_out/configs_${tag}.jsonl
ARGS="--steps 2 --warmup 3 --no-e2e --no-cpu-baseline --config 2 --fill 600"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:raas_decode -s $((600 * 4 * 32 + 1)) -c 16 --csv --log-file gpurun_out/launches_${tag}_cfg2.csv python bench.py $ARGS > /dev/null 2>&1; echo "cfg2 list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:raas_decode -s $((600 * 4 * 32 + 1)) -c 1 -o gpurun_out/prof_${tag}_cfg2 python bench.py $ARGS > /dev/null 2>&1; echo "cfg2 full rc=$?"
