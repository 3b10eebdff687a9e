O=gpurun_out/g63; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x > $O/tests.txt 2>&1; echo "rc=$?" >> $O/tests.txt
for i in 1 2; do
timeout 300 python tools/run_config.py c4 0 5 > $O/c4_$i.json 2>&1
H2G_JACOBI_CIRCLE=1 timeout 300 python tools/run_config.py c4 0 5 > $O/c4_circle_$i.json 2>&1
done
timeout 300 python tools/run_config.py c2 0 5 > $O/c2.json 2>&1
H2G_JACOBI_CIRCLE=1 timeout 300 python tools/run_config.py c2 0 5 > $O/c2_circle.json 2>&1
H2G_DEBUG_SWEEPS=1 H2G_SERIAL=1 timeout 300 python tools/run_config.py c4 0 1 > $O/sweeps_ring.txt 2>&1
timeout 600 ncu --kernel-name regex:svd_finish --metrics gpu__time_duration.sum --clock-control none --csv python tools/run_config.py c4 0 1 > $O/fin_ring.csv 2> /dev/null
H2G_JACOBI_CIRCLE=1 timeout 600 ncu --kernel-name regex:svd_finish --metrics gpu__time_duration.sum --clock-control none --csv python tools/run_config.py c4 0 1 > $O/fin_circle.csv 2> /dev/null
