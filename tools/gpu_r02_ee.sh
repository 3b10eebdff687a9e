O=gpurun_out/g58; mkdir -p $O
STAGES=1 timeout 600 python tools/step_loop.py c4 16 > $O/loop.txt 2>&1

