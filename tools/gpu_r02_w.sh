O=gpurun_out/g44; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q -x > $O/tests.txt 2>&1; echo "rc=$?" >> $O/tests.txt
for c in c4 c2; do timeout 300 python tools/run_config.py $c 0 5 > $O/${c}.json 2>&1; done
H2G_TRACE=$O/trace_c4.json timeout 300 python tools/trace_config.py c4 > $O/trace_c4.txt 2>&1
python tools/trace_summary.py $O/trace_c4.json > $O/trace_c4_summary.txt 2>&1; rm -f $O/trace_c4.json
