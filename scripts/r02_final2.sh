#!/bin/bash
# GPU box, round-2 closing evidence: the headline bench 5x (median), a whole 16k-step config-3
# run (prefill + 16384 decode steps of 32 layers, wall time incl. the GPU-drawn inputs), the
# configs table, and ncu of the L = 256 half-size-CTA kernel.
tag=${1:-r02z}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for i in 1 2 3 4 5; do timeout 900 python bench.py --no-cpu-baseline 2>/dev/null | tee -a gpurun_out/bench5_${tag}.jsonl | cut -c1-120; done
timeout 1800 python bench.py --fill 16384 --steps 20 --no-e2e --no-cpu-baseline 2> gpurun_out/wholerun_${tag}.log > gpurun_out/wholerun_${tag}.json; grep filled gpurun_out/wholerun_${tag}.log
bash scripts/run_configs.sh ${tag} > /dev/null 2>&1; wc -l gpurun_out/configs_${tag}.jsonl
ARGS="--steps 2 --warmup 3 --no-e2e --no-cpu-baseline --config 5 --L 256 --layers 8 --fill 200"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:raas_decode -s $((200 * 8 + 1)) -c 16 --csv --log-file gpurun_out/launches_${tag}_L256.csv python bench.py $ARGS > /dev/null 2>&1; echo "L256 list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:raas_decode -s $((200 * 8 + 1)) -c 1 -o gpurun_out/prof_${tag}_L256 python bench.py $ARGS > /dev/null 2>&1; echo "L256 full rc=$?"
timeout 900 python bench.py > gpurun_out/bench_${tag}.json 2> gpurun_out/bench_${tag}_stderr.log; cut -c1-200 gpurun_out/bench_${tag}.json
