#!/bin/bash
mkdir -p gpurun_out
bash scripts/sweep_variants.sh paper_2502_11147_b200/libraas.so build_exp/libraas_4388c6a.so build_exp/libraas_44c8f99.so build_exp/libraas_fcabae9.so build_exp/libraas_d44e054.so paper_2502_11147_b200/libraas.so build_exp/libraas_4388c6a.so
f=build_exp/libraas_4388c6a.so; n=$(basename $f .so)
RAAS_LIB=$f timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:raas_decode -s 60850 -c 32 --csv --log-file gpurun_out/launches_$n.csv python bench.py --fill 1900 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo "ncu $n rc=$?"
