#!/bin/bash
# GPU box: the other BASELINE.json configs (parity-test sizes are in tests/): config 2 (B=1,
# latency), config 4 (Qwen shapes), config 5 budget sweep + dense comparator.  JSON lines ->
# gpurun_out/configs_<tag>.jsonl
tag=${1:-dev}
out=gpurun_out/configs_${tag}.jsonl
mkdir -p gpurun_out; : > $out
run() { python bench.py "$@" --no-cpu-baseline 2>>gpurun_out/configs_${tag}.err | tee -a $out | cut -c1-200; }
run --config 2 --steps 200 --no-e2e
run --config 4 --steps 100 --no-e2e
for L in 256 512 1024 2048 4096 8192; do
  layers=4; [ $L -le 512 ] && layers=8
  run --config 5 --L $L --layers $layers --steps 100 --no-e2e
done
run --config 5 --dense 32896 --layers 4 --steps 20 --warmup 3 --no-e2e
# method variants at config 3 shapes
run --config 3 --steps 100 --no-e2e --score quest                 # NEXT-1 Quest bound stamps
run --config 3 --steps 100 --no-e2e --top-r 0.5                   # NEXT-3 top-r rule
run --config 3 --steps 100 --no-e2e --table-scope 1               # NEXT-2 one table per request
run --config 3 --steps 100 --no-e2e --page 1                      # NEXT-3 token level (deferred)
run --config 3 --steps 100 --no-e2e --P 1024                      # long prompt, plain RaaS
run --config 3 --steps 100 --no-e2e --P 1024 --quest-prefill 16   # NEXT-4 hybrid, K = 16
