O=gpurun_out/g30; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x > $O/tests.txt 2>&1; echo "rc=$?" >> $O/tests.txt
for c in c4 c2; do timeout 300 python tools/run_config.py $c 0 5 > $O/${c}.json 2>&1; H2G_NORM_CTA=1 timeout 300 python tools/run_config.py $c 0 5 > $O/${c}_cta.json 2>&1; done
timeout 600 ncu --kernel-name regex:norm_ --metrics gpu__time_duration.sum --clock-control none --csv \
  python tools/run_config.py c4 0 1 > $O/norm_launches_c4.csv 2> $O/norm_launches.err
