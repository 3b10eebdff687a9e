O=gpurun_out/g40; mkdir -p $O
H2G_DEBUG_MV=1 timeout 600 python tools/mv_debug.py c4 > $O/mv_debug.txt 2>&1
