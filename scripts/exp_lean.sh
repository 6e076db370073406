#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x 2>&1 | tail -3
bash scripts/sweep_variants.sh paper_2502_11147_b200/libraas.so build_exp/libraas_4388c6a.so paper_2502_11147_b200/libraas.so build_exp/libraas_4388c6a.so
