#!/bin/bash
# GPU box: parity tests, then the headline bench (stdout JSON -> gpurun_out/bench_<tag>.json)
tag=${1:-dev}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -25
python bench.py ${@:2} 2> gpurun_out/bench_${tag}_stderr.log | tee gpurun_out/bench_${tag}.json
tail -3 gpurun_out/bench_${tag}_stderr.log
