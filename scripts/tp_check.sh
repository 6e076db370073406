#!/bin/bash
# GPU box: tail-pool schedule checks (bitwise vs the default schedule, config 4 lockstep) and A/B
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "tail_pool or full_size_sampled or cluster_schedule or request_sharding" 2>&1 | tail -4
q() { RAAS_POOL=$1 timeout 600 python bench.py --no-e2e --no-cpu-baseline $2 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('pool=$1 | $2 |', round(d['roofline']['achieved']), 'GB/s |', round(d['roofline']['avg_launch_us'],2), 'us |', d['clocks']['sm_mhz'], 'MHz |', d['launch'])" || echo "pool=$1 | $2 | FAILED"; }
for rep in 1 2; do for f in 0 1; do
  q $f "--config 4 --steps 60"
  q $f "--config 3 --batch 8 --steps 100"
done; done 2>&1 | tee gpurun_out/tp_ab.txt
