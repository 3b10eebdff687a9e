mkdir -p gpurun_out/g19
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_stages.py -m gpu -q -x > gpurun_out/g19/tests.txt 2>&1; echo "rc=$?" >> gpurun_out/g19/tests.txt
for c in c4 c2 c3; do
timeout 300 python tools/run_config.py $c 0 5 > gpurun_out/g19/${c}.json 2>&1
H2G_PUSH_3F=1 timeout 300 python tools/run_config.py $c 0 5 > gpurun_out/g19/${c}_p3.json 2>&1
done
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/g19/launches_c4.csv 2> gpurun_out/g19/launches_c4.err
python tools/launch_summary.py gpurun_out/g19/launches_c4.csv 30 > gpurun_out/g19/launches_c4_summary.txt 2>&1
