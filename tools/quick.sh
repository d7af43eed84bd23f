#!/usr/bin/env bash
# quick GPU iteration: build, a parity subset, a short bench
cd "$(dirname "$0")/.."
python __graft_entry__.py > /dev/null 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 600 python -m pytest tests -m gpu -q -x --timeout 90 --timeout-method thread ${PYTEST_K:+-k "$PYTEST_K"} 2>&1 | tail -3
timeout 600 python bench.py --no-batch --no-cpu-baseline --steps 5 ${BENCH_ARGS:-} | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('value',round(d['value'],2),'ms/step',round(d['ms_per_step'],3),'breakdown',{k:round(v,3) for k,v in d['breakdown_ms'].items()},'frac',round(d['roofline']['frac'],4),'e2e',round(d['e2e']['value'],2))"
