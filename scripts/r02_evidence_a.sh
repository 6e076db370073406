#!/bin/bash
# GPU box, round-2 evidence part A: headline bench line, every config's line, kernel traces.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 900 python bench.py 2> gpurun_out/bench_r02_stderr.log > gpurun_out/bench_r02.json; cut -c1-300 gpurun_out/bench_r02.json
timeout 600 python bench.py --steps 20 --no-e2e --no-cpu-baseline --trace gpurun_out/trace_r02_cfg3.json > /dev/null 2>&1
timeout 600 python bench.py --config 4 --steps 20 --no-e2e --no-cpu-baseline --trace gpurun_out/trace_r02_cfg4.json > /dev/null 2>&1
timeout 600 python bench.py --config 2 --steps 20 --no-e2e --no-cpu-baseline --trace gpurun_out/trace_r02_cfg2.json > /dev/null 2>&1
for c in 3 4 2; do python scripts/trace_summary.py gpurun_out/trace_r02_cfg$c.json --layers 32 2>&1 | head -4; done
bash scripts/run_configs.sh r02
