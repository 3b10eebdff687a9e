O=gpurun_out/g60; mkdir -p $O
H2G_SERIAL=1 H2G_TRACE=$O/trace_c4_serial.json timeout 300 python tools/trace_config.py c4 > $O/trace_c4.txt 2>&1
