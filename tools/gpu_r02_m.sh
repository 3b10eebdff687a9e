O=gpurun_out/g24; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "matvec or golden_parity or estimate or live_oracle" > $O/tests.txt 2>&1; echo "rc=$?" >> $O/tests.txt
for c in c4 c2; do timeout 300 python tools/mv_bench.py $c > $O/mv_$c.json 2>&1; done
timeout 600 ncu --kernel-name regex:mv_ --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv \
  python tools/mv_bench.py c4 > $O/mv_launches_c4.csv 2> $O/mv_launches.err
