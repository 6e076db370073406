#!/bin/bash
# GPU box: full check = gpu tests, smoke, headline bench (JSON), other configs, ncu evidence.
tag=${1:-dev}
mkdir -p gpurun_out
python -m pytest tests -m gpu -q 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py 2> gpurun_out/bench_${tag}_stderr.log > gpurun_out/bench_${tag}.json; cat gpurun_out/bench_${tag}.json | cut -c1-400
bash scripts/run_configs.sh ${tag} > /dev/null
bash scripts/ncu_profile.sh ${tag}
