O=gpurun_out/g75; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/tests.txt 2>&1; echo "rc=$?" >> $O/tests.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "rc=$?" >> $O/smoke.txt
H2G_DEBUG_SWEEPS=1 timeout 600 python tools/run_config.py c4 0 1 > $O/sweeps_c4.txt 2>&1; echo "rc=$?" >> $O/sweeps_c4.txt
