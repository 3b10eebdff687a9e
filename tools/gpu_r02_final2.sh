# end-of-round check with the final library: full GPU suite, smoke, bench lines, launch list, trace, c5 at n = 131,072
O=gpurun_out/final2; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest.txt 2>&1; echo "pytest rc=$?" >> $O/pytest.txt; tail -3 $O/pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.txt 2>&1; tail -1 $O/smoke.txt
python bench.py --steps 10 --warmup 3 > $O/bench_c4.json 2> $O/bench_c4.err; echo "bench c4 rc=$?"
python bench.py --config c2 --steps 10 --warmup 3 > $O/bench_c2.json 2> $O/bench_c2.err; echo "bench c2 rc=$?"
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/launches_c4.csv 2> /dev/null; echo "launch list rc=$?"
python tools/launch_summary.py $O/launches_c4.csv 40 > $O/launches_c4_summary.txt
H2G_TRACE=$O/trace_c4.json python tools/trace_config.py c4 > /dev/null 2>&1
python tools/trace_summary.py $O/trace_c4.json > $O/trace_c4_summary.txt; rm -f $O/trace_c4.json
for c in c2 c3 c4; do python tools/run_config.py $c 0 5 > $O/full_$c.json 2> $O/full_$c.err; done
timeout 600 python tools/run_config.py c5 65536 5 > $O/full_c5_65536.json 2> $O/full_c5_65536.err; echo "c5 65536 rc=$?"
timeout 900 python tools/run_config.py c5 131072 3 > $O/full_c5_131072.json 2> $O/full_c5_131072.err; echo "c5 131072 rc=$?"
tail -c 600 $O/full_c5_131072.json
