mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 300 python scripts/sanitize_case.py 2>&1 | tail -2
timeout 1500 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/pytest_r02d.log 2>&1; tail -16 gpurun_out/pytest_r02d.log
for c in 0 1; do for rep in 1 2; do RAAS_CLUSTER=$c timeout 300 python bench.py --config 2 --steps 200 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cluster=$c', round(d['roofline']['avg_launch_us'],2), 'us', d['roofline']['kernel'][-40:], 'e2e', round(d['e2e']['value'],1), 'device', round(d['value'],1), d['config']['l2'][:60])"; done; done
timeout 600 python bench.py --steps 100 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg3', round(d['roofline']['avg_launch_us'],2), 'us e2e', round(d['e2e']['value'],1), 'device', round(d['value'],1))"
for L in 256 512; do timeout 600 python bench.py --config 5 --L $L --layers 8 --steps 100 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('L=$L', round(d['roofline']['avg_launch_us'],2), 'us', d['launch'])"; done
