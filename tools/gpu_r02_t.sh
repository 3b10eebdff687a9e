O=gpurun_out/g38; mkdir -p $O
H2G_DEBUG_SWEEPS=1 H2G_SERIAL=1 timeout 300 python tools/trace_config.py c4 > $O/sweeps_c4.txt 2>&1
