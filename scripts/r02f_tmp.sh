cp paper_2502_11147_b200/libraas.so build_exp/libraas_cur.so
python - <<'PY'
import os, sys
sys.path.insert(0, '.')
os.environ["RAAS_LIB"] = "build_exp/libraas_nc4s8m2.so"
from paper_2502_11147_b200.raas import RaasLayer
for (L, B, hq, hkv) in [(2048, 64, 32, 8), (4096, 32, 28, 4), (256, 64, 32, 8)]:
    print(L, B, RaasLayer(L, 1e-4, hq, hkv, 128, B).raas_launch_info())
PY
bash scripts/ab.sh "--steps 60;--config 4 --steps 40;--config 5 --L 256 --layers 8 --steps 100;--config 2 --steps 100" 2 build_exp/libraas_cur.so build_exp/libraas_nc4s8m2.so build_exp/libraas_nc4s8.so 2>&1 | grep "|"
