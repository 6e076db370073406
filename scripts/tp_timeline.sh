#!/bin/bash
# GPU box: in-stream timelines at config 4 (default vs tail-pool schedule), debug-timing build
mkdir -p gpurun_out
for pool in 0 1; do
  echo "== RAAS_POOL=$pool"
  RAAS_POOL=$pool TL_DUMP=gpurun_out/tl_c4_pool$pool.npy RAAS_LIB=build/dbg.so timeout 600 python scripts/timeline.py --B 32 --L 4096 --P 128 --Hq 28 --Hkv 4 --layers 8
done 2>&1 | tee gpurun_out/tp_timeline.txt
