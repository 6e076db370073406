#!/bin/bash
# GPU box, 1 GPU: the multi-rank paths of bench.py run end to end (ranks share the GPU over gloo;
# RAAS_BENCH_SHARE_GPU=1 lines are functional checks, not measurements)
export RAAS_BENCH_SHARE_GPU=1
for args in "--config 3 --steps 20 --layers 4 --no-cpu-baseline" "--config 2 --shard heads --steps 50 --no-cpu-baseline"; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
    bench.py --gpus 2 $args 2> gpurun_out/multirank_err.log | cut -c1-2000
  echo "rc=$?"
done
