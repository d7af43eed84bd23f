python __graft_entry__.py >/dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "schedule or weighted or critical or slicing or lflam or refine or memory or smoke or hub or chain" 2>&1 | tail -3
for o in 0 1; do PDNN_INDEXED_ITEMS=$o CFGS=4,8,3,2 timeout 300 python tools/step_probe.py | sed "s/^/ix=$o /"; done
PDNN_INDEXED_ITEMS=1 CFG=4 timeout 300 python tools/sweep_trace.py > gpurun_out/trace_ix1.json 2>&1
python -c "
import json;d=json.load(open('gpurun_out/trace_ix1.json'))
print('ix trace total',d['total_us'],'tl hopsum',d['tl']['hop_sum'],'bl hopsum',d['bl']['hop_sum'],'bl last', d['bl']['done_by_level_us'][-3:], 'tl last', d['tl']['done_by_level_us'][-2:])"
