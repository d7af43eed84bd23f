# ncu --set full of the kernels matching $K (regex) in one C4 bench step -> gpurun_out/prof_k.ncu-rep
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$K" -c ${C:-2} \
  -o gpurun_out/prof_k -f python bench.py --steps 1 --warmup 0 --no-batch --no-cpu-baseline ${BENCH_ARGS:-} > gpurun_out/ncu_k.log 2>&1; echo "ncu rc=$?"
