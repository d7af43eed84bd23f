# run the quick bench once per value of an env var:  VAR=PDNN_SORT_FLAGS VALS="0 1 2" bash tools/sweep_env.sh
cd "$(dirname "$0")/.."
python __graft_entry__.py > /dev/null 2>&1 || { echo BUILD FAILED; exit 1; }
for v in $VALS; do
  echo "== $VAR=$v"
  env $VAR=$v timeout 300 python bench.py --no-batch --no-cpu-baseline --steps ${STEPS:-5} ${BENCH_ARGS:-} | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('value',round(d['value'],2),'ms/step',round(d['ms_per_step'],3),'breakdown',{k:round(v,3) for k,v in d['breakdown_ms'].items()},'frac',round(d['roofline']['frac'],4))"
done
