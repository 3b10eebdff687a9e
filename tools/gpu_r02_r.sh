O=gpurun_out/g33; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "golden_parity" > $O/tests.txt 2>&1; echo "rc=$?" >> $O/tests.txt
timeout 600 ncu --kernel-name regex:norm_lz_kernel --launch-skip 2 --launch-count 1 --set full --import-source on --clock-control none \
  -o $O/norm_lz -f python tools/run_config.py c4 0 1 > $O/norm_lz.log 2>&1
ncu -i $O/norm_lz.ncu-rep --page raw --csv > $O/norm_lz_raw.csv 2>/dev/null
python tools/ncu_stalls.py $O/norm_lz.ncu-rep norm_lz 40 > $O/norm_lz_stalls.txt 2>&1
timeout 300 python tools/run_config.py c4 0 5 > $O/c4.json 2>&1
