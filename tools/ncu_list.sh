#!/usr/bin/env bash
# per-kernel device times of one bench step (ncu launch list), summarised
cd "$(dirname "$0")/.."
python __graft_entry__.py > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-batch --no-cpu-baseline ${BENCH_ARGS:-} > /dev/null 2>&1
python tools/summarize_launches.py gpurun_out/launches.csv
