O=gpurun_out/g67; mkdir -p $O
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/run_config.py c5 65536 1 > $O/launches_c5.csv 2> /dev/null
python tools/launch_summary.py $O/launches_c5.csv 30 > $O/launches_c5_summary.txt 2>&1
H2G_TRACE=$O/trace_c5.json timeout 600 python tools/trace_config.py c5 65536 > $O/trace_c5.txt 2>&1
python tools/trace_summary.py $O/trace_c5.json > $O/trace_c5_summary.txt 2>&1; rm -f $O/trace_c5.json
