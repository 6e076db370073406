#!/bin/bash
# GPU box: the whole GPU test suite, smoke(), the headline line and every config's line.
tag=${1:-r02}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 2400 python -m pytest tests -m gpu -q --durations=12 > gpurun_out/pytest_${tag}.log 2>&1; tail -16 gpurun_out/pytest_${tag}.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py 2> gpurun_out/bench_${tag}_stderr.log > gpurun_out/bench_${tag}.json; cut -c1-200 gpurun_out/bench_${tag}.json
bash scripts/run_configs.sh ${tag} > /dev/null 2>&1; wc -l gpurun_out/configs_${tag}.jsonl
