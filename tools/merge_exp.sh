#!/usr/bin/env bash
# item merge order experiment (debug library knobs read at graph build)
cd "$(dirname "$0")/.."
python __graft_entry__.py > /dev/null 2>&1
for m in ${MODES:-0 1}; do
  PDNN_MERGE_MODE=$m CFGS=${CFGS:-2,3,4,6,8} timeout 300 python tools/sweep_probe.py | sed "s/^/merge=$m /"
  PDNN_MERGE_MODE=$m CFG=4 timeout 300 python tools/sweep_trace.py > gpurun_out/trace_m$m.json 2>&1
  python -c "
import json;d=json.load(open('gpurun_out/trace_m$m.json'))
print('merge=$m trace total',d['total_us'],'tl hopsum',d['tl']['hop_sum'],'bl hopsum',d['bl']['hop_sum'],'bl last', d['bl']['done_by_level_us'][-3:], 'tl last', d['tl']['done_by_level_us'][-2:])"
done
for m in ${MODES:-0 1}; do
  echo "batched bmerge=$m"; PDNN_DBG=1 PDNN_BMERGE_MODE=$m BS=${BS:-512,4096} timeout 300 python tools/batch_probe.py
done
