#!/usr/bin/env bash
# build, full GPU parity suite, single-sweep probes (C2-C4), batched probes
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail gpurun_out/build.log; exit 1; }
if [ "${TESTS:-1}" = "1" ]; then timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 2>&1 | tail -4; fi
for c in 2 3 4; do CFG=$c timeout 300 python tools/sweep_probe.py 2>&1 | tail -1 | cut -c1-110; done
PDNN_BATCH_NO_MEM=1 BS=${BS:-32,1024,4096} timeout 300 python tools/batch_probe.py 2>&1 | tail -3
