O=gpurun_out/g71; mkdir -p $O
H2G_DEBUG_MEM=1 timeout 300 python tools/debug_mem.py c2 > $O/mem_single.txt 2>&1
MEM0=1 timeout 600 python tools/debug_shard.py c2_full > $O/mem_p2.txt 2>&1
