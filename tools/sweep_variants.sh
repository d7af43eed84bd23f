#!/usr/bin/env bash
# compile-time variants of the sweep, timed by tools/sweep_probe.py (GPU box)
cd "$(dirname "$0")/.."
python __graft_entry__.py > /dev/null 2>&1
for v in "${@}"; do
  name="${v%%:*}"; defs="${v#*:}"
  VARIANT="_$name" DEFS="$defs" CFGS=${CFGS:-2,3,4} VARIANTS="${VARIANTS:-base;PDNN_SWEEP_NOWAIT=1}" timeout 300 python tools/sweep_probe.py
done
