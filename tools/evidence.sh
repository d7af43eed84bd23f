#!/usr/bin/env bash
# One GPU pass that regenerates the judged evidence (round R, default r2):
# bench line, ncu launch lists (C4 single-graph step, C5 batched evaluation),
# --set full captures of the hot kernels, the sweep's per-item trace.
# Outputs land in gpurun_out/ (summaries are copied to profiles/ by hand).
set -u
cd "$(dirname "$0")/.."
R=${R:-r2}
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 1200 python bench.py > gpurun_out/${R}_bench.json 2> gpurun_out/${R}_bench.err; echo "bench rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${R}_launches_c4.csv \
    python bench.py --steps 2 --warmup 1 --no-batch --no-cpu-baseline --no-shapes > /dev/null 2>&1; echo "ncu c4 list rc=$?"
BS=4096 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${R}_launches_c5.csv \
    python tools/batch_probe.py > /dev/null 2>&1; echo "ncu c5 list rc=$?"
# the timed step's kernels (warm-up step skipped)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_sweep|k_mem|k_cp|k_labels" -s 8 -c 8 \
    -o gpurun_out/${R}_prof_c4 -f python bench.py --steps 1 --warmup 1 --no-batch --no-cpu-baseline --no-shapes > gpurun_out/ncu_c4.log 2>&1; echo "ncu c4 full rc=$?"
BS=1024 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_bsweep|k_mem_sort|k_mem_edges|k_mem_scan|k_bcp" -c 5 \
    -o gpurun_out/${R}_prof_c5 -f python tools/batch_probe.py > gpurun_out/ncu_c5.log 2>&1; echo "ncu c5 full rc=$?"
CFG=4 timeout 300 python tools/sweep_trace.py > gpurun_out/${R}_sweep_trace_c4.json 2>&1; echo "trace rc=$?"
# NEXT-row probes (LFLAM, refinement) and the build phases
timeout 900 python tools/lflam_probe.py 2 6 3 4 > gpurun_out/${R}_lflam_probe.log 2>&1; echo "lflam probe rc=$?"
timeout 900 python tools/refine_probe.py 6 2 3 > gpurun_out/${R}_refine_probe.log 2>&1; echo "refine probe rc=$?"
CFGS=2,3,4,7 timeout 300 python tools/build_probe.py > gpurun_out/${R}_build_probe.log 2>&1; echo "build probe rc=$?"
