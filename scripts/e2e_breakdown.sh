#!/bin/bash
# GPU box: e2e (host-buffer API) vs device figure, A/B of libraas builds (RAAS_LIB), 2 reps each;
# RAAS_DBG_E2E builds: mode 1 = out to device (no host writes), 2 = no ingest (stale inputs)
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
for rep in 1 2; do for lib in "$@"; do
RAAS_LIB=$lib timeout 600 python bench.py --no-cpu-baseline --steps 100 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$(basename $lib) e2e', round(d['e2e']['value'],1), 'dev', round(d['value'],1), d['clocks']['sm_mhz'])"
done; done
