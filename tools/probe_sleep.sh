cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1
for sl in 0 100 -1000 -4000; do echo "bsleep $sl"; PDNN_BPOLL_SLEEP_NS=$sl PDNN_BATCH_NO_MEM=1 BS=32,1024 timeout 300 python tools/batch_probe.py 2>&1 | tail -2; done
for sl in 0 100 -1000; do for c in 3 4; do echo "single sleep $sl cfg $c"; CFG=$c PDNN_POLL_SLEEP_NS=$sl timeout 300 python tools/sweep_probe.py 2>&1 | tail -1 | cut -c1-120; done; done
