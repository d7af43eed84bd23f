set -u
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { echo BUILD FAIL; tail gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests -m gpu -q -x -k "weighted or critical or slicing or eval_batch or refine or hub or chain or lflam" 2>&1 | tail -3
for o in 1 0; do PDNN_BL_READY_ORDER=$o CFG=4 timeout 300 python tools/sweep_trace.py > gpurun_out/trace_c4_o$o.json 2>&1; echo "trace $o rc=$?"; done
timeout 600 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/bench3.json 2> gpurun_out/bench3.err; echo "bench rc=$?"
python - <<'P'
import json
d=json.loads(open('gpurun_out/bench3.json').read().strip().splitlines()[-1])
print('value',d['value'],'ms',d['ms_per_step'],'bd',d['breakdown_ms'],'frac',d['roofline']['frac'])
b=d.get('batched',{}); print('batched',b.get('value'),b.get('refine_evals_s'),b.get('projection_1gpu'))
for k,v in d.get('shapes',{}).items(): print(k, v.get('ms_per_step'), v.get('sweep_ms'), v.get('GTEPS'))
P
for o in 1 0; do python -c "
import json;d=json.load(open('gpurun_out/trace_c4_o$o.json'))
print('o=$o total',d['total_us'],'tl hopsum',d['tl']['hop_sum'],'bl hopsum',d['bl']['hop_sum'])
print(' bl done', d['bl']['done_by_level_us'][-12:])
print(' tl done', d['tl']['done_by_level_us'][-6:])
"; done
timeout 900 python tools/refine_probe.py 6 2 3 2>&1 | tail -4
