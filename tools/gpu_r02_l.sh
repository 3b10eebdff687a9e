# Session baseline: full GPU suite, c4/c2 product times, trace split and launch list of HEAD.
O=gpurun_out/g20; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest.txt 2>&1; echo "pytest rc=$?" >> $O/pytest.txt
for c in c4 c2 c3; do timeout 300 python tools/run_config.py $c 0 5 > $O/${c}.json 2>&1; done
H2G_TRACE=$O/trace_c4.json timeout 300 python tools/trace_config.py c4 > $O/trace_c4.txt 2>&1
python tools/trace_summary.py $O/trace_c4.json > $O/trace_c4_summary.txt 2>&1; rm -f $O/trace_c4.json
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/launches_c4.csv 2> $O/launches_c4.err
python tools/launch_summary.py $O/launches_c4.csv 40 > $O/launches_c4_summary.txt 2>&1
