cd $GRAFT_REPO_ROOT; python __graft_entry__.py > /dev/null 2>&1
for sl in 0 64 256 -512; do echo "bsleep $sl"; PDNN_BPOLL_SLEEP_NS=$sl PDNN_BATCH_NO_MEM=1 BS=32,256,4096 timeout 300 python tools/batch_probe.py 2>&1 | tail -3; done
BS=256,1024 timeout 300 python tools/batch_probe.py 2>&1 | tail -2
