#!/bin/bash
# e2e (host API) A/B of alternative builds at config 3
q() { RAAS_LIB=$1 python bench.py --no-cpu-baseline "${@:2}" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$(basename $1 .so)', '${*:2}', 'device', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), d['clocks']['sm_mhz'])"; }
for rep in 1 2 3; do for f in "$@"; do q $f --steps 100; done; done
