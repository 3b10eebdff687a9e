O=gpurun_out/g45; mkdir -p $O
H2G_DEBUG_ALLOC=1 H2G_DEBUG_MEM=1 timeout 300 python tools/run_config.py c4 0 3 > $O/c4_alloc.txt 2>&1
H2G_SYNC_EXPAND=1 H2G_DEBUG_ALLOC=1 H2G_DEBUG_MEM=1 timeout 300 python tools/run_config.py c4 0 3 > $O/c4_alloc_sync.txt 2>&1
