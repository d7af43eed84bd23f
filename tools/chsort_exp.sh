#!/usr/bin/env bash
# chunked-sort grid experiment: CTAs per SM of the single-placement sort
cd "$(dirname "$0")/.."
python __graft_entry__.py > /dev/null 2>&1
for b in 2 1; do
  echo "ch_bpsm=$b"; PDNN_CH_BPSM=$b CFGS=${CFGS:-3,4} timeout 300 python tools/mem_probe.py
done
