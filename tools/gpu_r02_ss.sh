O=gpurun_out/g73; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "golden_parity" > $O/tests.txt 2>&1; echo "rc=$?" >> $O/tests.txt
for L in 128 64; do
H2G_CHOL_256=$L timeout 300 python tools/run_config.py c4 0 5 > $O/c4_$L.json 2>&1
H2G_CHOL_256=$L timeout 600 ncu --kernel-name regex:gram_chol --metrics gpu__time_duration.sum --clock-control none --csv python tools/run_config.py c4 0 1 > $O/chol_$L.csv 2> /dev/null
done
