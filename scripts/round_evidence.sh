#!/bin/bash
# GPU box, end of round: parity suite, smoke, headline bench line, the other configs and
# variants, ncu launch lists + full captures (config 3, config 4, config 5 L=256 / L=8192)
tag=${1:-r01}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -3 | tee gpurun_out/tests_${tag}.txt
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1 | tee gpurun_out/smoke_${tag}.txt
python bench.py 2> gpurun_out/bench_${tag}_stderr.log > gpurun_out/bench_${tag}.json; cut -c1-300 gpurun_out/bench_${tag}.json
bash scripts/run_configs.sh ${tag} > /dev/null
bash scripts/ncu_profile.sh ${tag}
bash scripts/ncu_configs.sh ${tag}
