O=gpurun_out/g76; mkdir -p $O
bash tools/ab.sh paper_2309_09061_b200/libh2g.so build_ab/libh2g_unroll.so 3 > $O/ab.txt 2>&1
