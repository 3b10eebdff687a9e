O=gpurun_out/g61; mkdir -p $O
timeout 900 python tools/e2e_split_c4.py c4 > $O/e2e_split.txt 2>&1
