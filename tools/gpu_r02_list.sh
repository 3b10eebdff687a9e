O=gpurun_out/list; mkdir -p $O
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/launches_c4.csv 2> /dev/null; echo "launch list rc=$?"
python tools/launch_summary.py $O/launches_c4.csv 60 > $O/launches_c4_summary.txt
H2G_TRACE=$O/trace_c4.json python tools/trace_config.py c4 > /dev/null 2>&1
python tools/trace_summary.py $O/trace_c4.json > $O/trace_c4_summary.txt; rm -f $O/trace_c4.json
head -24 $O/launches_c4_summary.txt
