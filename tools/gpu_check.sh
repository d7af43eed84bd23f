#!/usr/bin/env bash
# One GPU-box pass: tests with durations, the bench, the ncu launch list and
# `--set full` captures of the hot kernels.  Outputs land in gpurun_out/.
#   TESTS=0 skips pytest, NCU=0 skips ncu, BENCH_ARGS passes bench flags.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1
if [ "${TESTS:-1}" = "1" ]; then
  timeout 900 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
  tail -25 gpurun_out/pytest_gpu.log
fi
timeout 900 python bench.py ${BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
cat gpurun_out/bench.json; tail -5 gpurun_out/bench.err
if [ "${NCU:-1}" = "1" ]; then
  NB="--no-batch --no-cpu-baseline"
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
      python bench.py --steps 2 --warmup 1 $NB > gpurun_out/ncu_launch_bench.log 2>&1; echo "ncu list rc=$?"
  timeout 900 ncu --set full --clock-control none --import-source on \
      -k regex:"k_sweep|k_mem_edges|k_mem_scan|k_cp|k_mem_prep|k_mem_sort_chunk" -c 7 \
      -o gpurun_out/prof_full -f python bench.py --steps 1 --warmup 0 $NB \
      > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
  # the visit-order sort of the memory scan: skip the graph build's sorts
  timeout 900 ncu --set full --clock-control none -k regex:"Onesweep" -s ${SORT_SKIP:-30} -c 3 \
      -o gpurun_out/prof_sort -f python bench.py --steps 1 --warmup 0 $NB \
      > gpurun_out/ncu_sort.log 2>&1; echo "ncu sort rc=$?"
fi
