cp paper_2502_11147_b200/libraas.so build_exp/libraas_cur.so
bash scripts/ab.sh "--config 2 --steps 200;--steps 60;--config 4 --steps 40;--config 5 --L 256 --layers 8 --steps 100" 2 build_exp/libraas_cur.so build_exp/libraas_pre16.so 2>&1 | grep "|"
