#!/usr/bin/env bash
# One GPU pass that regenerates the judged evidence: bench line, ncu launch
# lists (C4 single-graph step, C5 batched evaluation) and --set full captures
# of the hot kernels.  Outputs land in gpurun_out/ (copy summaries to profiles/).
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv \
    python bench.py --steps 2 --warmup 1 --no-batch --no-cpu-baseline > /dev/null 2>&1; echo "ncu c4 list rc=$?"
BS=4096 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5.csv \
    python tools/batch_probe.py > /dev/null 2>&1; echo "ncu c5 list rc=$?"
# placement-aware sweep of the bench step = the 3rd k_sweep launch (warm-up step: slice + placement)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_sweep|k_mem_sort_chunk|k_mem_edges|k_mem_scan|k_cp|k_mem_prep|k_labels" -s 9 -c 9 \
    -o gpurun_out/prof_c4 -f python bench.py --steps 1 --warmup 1 --no-batch --no-cpu-baseline > gpurun_out/ncu_c4.log 2>&1; echo "ncu c4 full rc=$?"
BS=1024 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_bsweep|k_mem_sort|k_mem_edges|k_mem_scan|k_bcp" -c 5 \
    -o gpurun_out/prof_c5 -f python tools/batch_probe.py > gpurun_out/ncu_c5.log 2>&1; echo "ncu c5 full rc=$?"
