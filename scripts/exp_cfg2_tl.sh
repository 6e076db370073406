#!/bin/bash
# config 2 (B = 1, L = 1024): in-stream timelines (RAAS_DBG_TIMING build), graph and eager
export RAAS_LIB=build_exp/libraas_dbg.so
python scripts/timeline.py --B 1 --L 1024 --P 512 --sp 16
python scripts/timeline.py --B 1 --L 1024 --P 512 --sp 16 --graph 0
python scripts/timeline.py --B 1 --L 1024 --P 512 --sp 32
RAAS_GRID=8 python scripts/timeline.py --B 1 --L 1024 --P 512 --sp 32
