#!/usr/bin/env bash
# bl items by their readiness wave (PDNN_BL_READY_ORDER=1) vs by level (0)
cd "$(dirname "$0")/.."
python __graft_entry__.py > /dev/null 2>&1
for o in 0 1; do
  PDNN_BL_READY_ORDER=$o CFGS=${CFGS:-3,4,2,6,8} timeout 300 python tools/step_probe.py | sed "s/^/blr=$o /"
  echo "batched blr=$o"; PDNN_DBG=1 PDNN_BL_READY_ORDER=$o BS=${BS:-512,4096} timeout 300 python tools/batch_probe.py
done
