#!/usr/bin/env bash
# compile-time variants of the memory tracker, timed by tools/mem_probe.py (GPU box)
#   bash tools/mem_variants.sh "name:DEF1=1 DEF2=2" ...
cd "$(dirname "$0")/.."
python __graft_entry__.py > /dev/null 2>&1
for v in "${@}"; do
  name="${v%%:*}"; defs="${v#*:}"
  VARIANT="_$name" DEFS="$defs" CFGS=${CFGS:-3,4} timeout 300 python tools/mem_probe.py
done
if [ "${BATCH:-0}" = "1" ]; then
  for v in "${@}"; do
    name="${v%%:*}"; defs="${v#*:}"
    echo "batch $name"; VARIANT="_$name" DEFS="$defs" BS=${BS:-1024,4096} timeout 300 python tools/batch_probe.py
  done
fi
