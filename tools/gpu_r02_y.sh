O=gpurun_out/g53; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x > $O/tests.txt 2>&1; echo "rc=$?" >> $O/tests.txt
for c in c4 c2; do timeout 300 python tools/run_config.py $c 0 5 > $O/${c}.json 2>&1; done
timeout 600 ncu --kernel-name regex:gram_ --metrics gpu__time_duration.sum --clock-control none --csv python tools/run_config.py c4 0 1 > $O/gram_launches_c4.csv 2> /dev/null
