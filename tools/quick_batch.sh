#!/usr/bin/env bash
# GPU iteration for the batched path: build, batch parity, probe timings
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests -m gpu -q -x --timeout 300 ${PYTEST_K:+-k "$PYTEST_K"} 2>&1 | tail -15
PDNN_BATCH_NO_MEM=1 BS=${BS:-32,256,1024,4096} timeout 300 python tools/batch_probe.py 2>&1 | tail -8
BS=${BS2:-32,256} timeout 300 python tools/batch_probe.py 2>&1 | tail -4
