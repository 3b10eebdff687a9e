O=gpurun_out/g31; mkdir -p $O
timeout 300 python tools/norm_check.py c4 > $O/norm_lz.txt 2>&1
H2G_NORM_CTA=1 timeout 300 python tools/norm_check.py c4 > $O/norm_cta.txt 2>&1
