#!/bin/bash
# GPU box: every BASELINE.json config beside the headline (parity-test sizes are in tests/):
# config 2 (B = 1, latency; cluster schedule), config 4 (Qwen shapes), config 5 budget sweep +
# dense comparator, the strong-scaling shards (what each of G request-sharded ranks runs: no
# collective, so G ranks take max over ranks of these), and the method variants.
# JSON lines -> gpurun_out/configs_<tag>.jsonl
tag=${1:-dev}
out=gpurun_out/configs_${tag}.jsonl
mkdir -p gpurun_out; : > $out
run() { timeout 900 python bench.py "$@" --no-cpu-baseline 2>>gpurun_out/configs_${tag}.err | tee -a $out | cut -c1-160; }
run --config 2 --steps 200
run --config 4 --steps 100 --no-e2e
for L in 256 512 1024 2048 4096 8192; do
  layers=4; [ $L -le 512 ] && layers=8
  run --config 5 --L $L --layers $layers --steps 100 --no-e2e
done
run --config 5 --dense 32896 --layers 4 --steps 20 --warmup 3 --no-e2e
# strong-scaling shards: config 4's global 256 requests over G = 1 / 2 / 4 (G = 8 is the weak
# line above), config 3's global 64 over G = 2 / 4 / 8
for B in 256 128 64; do run --config 4 --batch $B --steps 60 --no-e2e; done
for B in 32 16 8; do run --config 3 --batch $B --steps 100 --no-e2e; done
# method variants at config 3 shapes
run --config 3 --steps 100 --no-e2e --score quest                 # NEXT-1 Quest bound stamps
run --config 3 --steps 100 --no-e2e --top-r 0.5                   # NEXT-3 top-r rule
run --config 3 --steps 100 --no-e2e --table-scope 1               # NEXT-2 one table per request
run --config 3 --steps 100 --no-e2e --page 1                      # NEXT-3 token level (deferred)
run --config 3 --steps 100 --no-e2e --P 1024                      # long prompt, plain RaaS
run --config 3 --steps 100 --no-e2e --P 1024 --quest-prefill 16   # NEXT-4 hybrid, K = 16
