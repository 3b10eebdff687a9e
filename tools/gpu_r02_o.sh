O=gpurun_out/g29; mkdir -p $O
H2G_TRACE=$O/trace_c4.json timeout 300 python tools/trace_config.py c4 > $O/trace_c4.txt 2>&1
python tools/trace_summary.py $O/trace_c4.json > $O/trace_c4_summary.txt 2>&1
python tools/trace_summary.py $O/trace_c4.json 2 > $O/trace_c4_s2.txt 2>&1
rm -f $O/trace_c4.json
