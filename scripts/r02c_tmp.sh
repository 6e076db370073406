mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_r02c.log 2>&1; tail -4 gpurun_out/pytest_r02c.log
cp paper_2502_11147_b200/libraas.so build_exp/libraas_cl.so
bash scripts/ab.sh "--config 2 --steps 200;--steps 60" 2 build_exp/libraas_cl.so build_exp/libraas_nocl.so 2>&1 | grep "|" | tee gpurun_out/ab_r02c.txt
for f in build_exp/libraas_cl.so build_exp/libraas_nocl.so; do for rep in 1 2; do RAAS_LIB=$f timeout 600 python bench.py --steps 60 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$f e2e', round(d['e2e']['value'],1), 'device', round(d['value'],1))"; done; done | tee -a gpurun_out/ab_r02c.txt
RAAS_CLUSTER=0 timeout 600 python bench.py --config 2 --steps 200 --no-cpu-baseline --no-e2e 2>/dev/null | cut -c1-120
