set -u
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_mem" -c 8 \
  -o gpurun_out/prof_mem -f python bench.py --steps 1 --warmup 0 --no-batch --no-cpu-baseline > gpurun_out/ncu_mem.log 2>&1; echo "ncu rc=$?"
