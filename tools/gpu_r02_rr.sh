O=gpurun_out/g72; mkdir -p $O
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench_c4.json 2> $O/bench_c4.err; echo "rc=$?" >> $O/bench_c4.err
timeout 600 python bench.py --config c2 --steps 10 --warmup 3 > $O/bench_c2.json 2> $O/bench_c2.err
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/launches_c4.csv 2> $O/launches_c4.err
python tools/launch_summary.py $O/launches_c4.csv 40 > $O/launches_c4_summary.txt 2>&1
H2G_TRACE=$O/trace_c4.json timeout 300 python tools/trace_config.py c4 > $O/trace_c4.txt 2>&1
python tools/trace_summary.py $O/trace_c4.json > $O/trace_c4_summary.txt 2>&1; rm -f $O/trace_c4.json
