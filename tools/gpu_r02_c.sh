mkdir -p gpurun_out/g4
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x > gpurun_out/g4/tests.txt 2>&1; echo "rc=$?" >> gpurun_out/g4/tests.txt
timeout 300 python tools/run_config.py c4 0 3 > gpurun_out/g4/c4.json 2>&1
H2G_SERIAL=1 H2G_TRACE=gpurun_out/g4/trace_c4_serial.json timeout 300 python tools/trace_config.py c4 > gpurun_out/g4/trace_c4_serial.txt 2>&1
python tools/trace_summary.py gpurun_out/g4/trace_c4_serial.json > gpurun_out/g4/trace_c4_serial_summary.txt 2>&1
rm -f gpurun_out/g4/trace_c4_serial.json
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/g4/launches_c4.csv 2> gpurun_out/g4/launches_c4.err
python tools/launch_summary.py gpurun_out/g4/launches_c4.csv 40 > gpurun_out/g4/launches_c4_summary.txt 2>&1
