#!/bin/bash
# GPU box: the GPU test suite (durations), smoke(), then the headline bench line.
# usage: scripts/gpu_check.sh <tag> [pytest -k expr] [bench args...]
tag=${1:-dev}; kexpr=${2:-}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_${tag}.log 2>&1 || tail -20 gpurun_out/build_${tag}.log
if [ -n "$kexpr" ]; then
  timeout 3000 python -m pytest tests -m gpu -q --durations=15 -k "$kexpr" > gpurun_out/pytest_${tag}.log 2>&1
else
  timeout 3000 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/pytest_${tag}.log 2>&1
fi
tail -40 gpurun_out/pytest_${tag}.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py ${@:3} 2> gpurun_out/bench_${tag}_stderr.log > gpurun_out/bench_${tag}.json
tail -2 gpurun_out/bench_${tag}_stderr.log; cut -c1-600 gpurun_out/bench_${tag}.json
