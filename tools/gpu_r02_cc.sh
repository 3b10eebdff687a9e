O=gpurun_out/g54; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_stages.py -m gpu -q -x > $O/tests.txt 2>&1; echo "rc=$?" >> $O/tests.txt
for c in c4 c2; do timeout 300 python tools/run_config.py $c 0 5 > $O/${c}.json 2>&1; done
H2G_GSUM_NO_SMALL=1 timeout 300 python tools/run_config.py c4 0 5 > $O/c4_nosmall.json 2>&1
timeout 600 ncu --kernel-name regex:gsum --metrics gpu__time_duration.sum --clock-control none --csv python tools/run_config.py c4 0 1 > $O/gsum_launches_c4.csv 2> /dev/null
