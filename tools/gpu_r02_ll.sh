O=gpurun_out/g66; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x > $O/tests.txt 2>&1; echo "rc=$?" >> $O/tests.txt
timeout 600 python tools/run_config.py c5 65536 5 > $O/c5.json 2>&1
timeout 300 python tools/run_config.py c4 0 5 > $O/c4.json 2>&1
H2G_DEBUG_SWEEPS=1 H2G_SERIAL=1 timeout 600 python tools/run_config.py c5 65536 1 > $O/sweeps_c5.txt 2>&1
