#!/usr/bin/env bash
# One GPU-box pass: tests with durations, the bench, the ncu launch list and
# one `--set full` capture of the hot kernels.  Outputs land in gpurun_out/.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -25 gpurun_out/pytest_gpu.log
timeout 600 python bench.py ${BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
cat gpurun_out/bench.json; tail -5 gpurun_out/bench.err
if [ "${NCU:-1}" = "1" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
      python bench.py --steps 2 --warmup 1 --no-batch --no-cpu-baseline > gpurun_out/ncu_launch_bench.log 2>&1; echo "ncu list rc=$?"
  timeout 900 ncu --set full --clock-control none --import-source on \
      -k regex:"k_sweep|Onesweep|k_mem_edges|k_mem_tile_final|k_cp|k_mem_prep" -c 8 \
      -o gpurun_out/prof_full -f python bench.py --steps 1 --warmup 0 --no-batch --no-cpu-baseline \
      > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
fi
