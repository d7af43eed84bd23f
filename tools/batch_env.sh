# batched probe once per value of an env var:  VAR=PDNN_BPOLL_SLEEP_NS VALS="0 100" BS=512,4096 bash tools/batch_env.sh
cd "$(dirname "$0")/.."
python __graft_entry__.py > /dev/null 2>&1 || { echo BUILD FAILED; exit 1; }
for v in $VALS; do
  echo "== $VAR=$v"
  env $VAR=$v PDNN_BATCH_NO_MEM=${NO_MEM:-} BS=${BS:-512,4096} timeout 300 python tools/batch_probe.py
done
