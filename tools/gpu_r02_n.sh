O=gpurun_out/g28; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "matvec or golden_parity or estimate or live_oracle" > $O/tests.txt 2>&1; echo "rc=$?" >> $O/tests.txt
for c in c4 c2; do timeout 300 python tools/mv_bench.py $c > $O/mv_$c.json 2>&1; done
O=gpurun_out/g28; mkdir -p $O
timeout 600 ncu --kernel-name regex:mv_warp_kernel --launch-skip 6 --launch-count 1 --set full --import-source on --clock-control none \
  -o $O/mv_coup -f python tools/mv_bench.py c4 > $O/mv_coup.log 2>&1
ncu -i $O/mv_coup.ncu-rep --page source --csv > $O/mv_coup_src.csv 2>/dev/null
ncu -i $O/mv_coup.ncu-rep --page raw --csv > $O/mv_coup_raw.csv 2>/dev/null
python tools/ncu_stalls.py $O/mv_coup.ncu-rep mv_warp 40 > $O/mv_coup_stalls.txt 2>&1
