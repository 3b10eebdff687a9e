O=gpurun_out/g41; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stages.py -m gpu -q -x > $O/tests.txt 2>&1; echo "rc=$?" >> $O/tests.txt
for c in c4 c2; do timeout 300 python tools/run_config.py $c 0 5 > $O/${c}.json 2>&1; done
H2G_TRACE=$O/trace_c4.json timeout 300 python tools/trace_config.py c4 > $O/trace_c4.txt 2>&1
python tools/trace_summary.py $O/trace_c4.json > $O/trace_c4_summary.txt 2>&1; rm -f $O/trace_c4.json
timeout 600 ncu --kernel-name regex:norm_ --metrics gpu__time_duration.sum --clock-control none --csv python tools/run_config.py c4 0 1 > $O/norm_launches_c4.csv 2> /dev/null
