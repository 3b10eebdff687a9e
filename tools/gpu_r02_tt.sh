O=gpurun_out/g74; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/tests.txt 2>&1; echo "rc=$?" >> $O/tests.txt
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench_c4.json 2> $O/bench_c4.err; echo "rc=$?" >> $O/bench_c4.err
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "rc=$?" >> $O/smoke.txt
