cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/pingpong tools/micro/pingpong.cu && /tmp/pingpong > gpurun_out/pingpong.txt 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/gather tools/micro/gather.cu && /tmp/gather > gpurun_out/gather.txt 2>&1
for c in 4 3 2; do CFG=$c PDNN_SWEEP_STATS=1 timeout 300 python tools/sweep_probe.py >> gpurun_out/probe.txt 2>&1; CFG=$c timeout 300 python tools/sweep_probe.py >> gpurun_out/probe.txt 2>&1; done
nvidia-smi -q | grep -i -A3 "Max Clocks" > gpurun_out/smi.txt
