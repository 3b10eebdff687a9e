mkdir -p gpurun_out/g3
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x > gpurun_out/g3/tests.txt 2>&1; echo "rc=$?" >> gpurun_out/g3/tests.txt
for v in new v1; do
  if [ $v = v1 ]; then export H2G_GSUM_V1=1; fi
  timeout 300 python tools/run_config.py c4 0 3 > gpurun_out/g3/c4_$v.json 2>&1
  timeout 300 python tools/run_config.py c2 0 5 > gpurun_out/g3/c2_$v.json 2>&1
  H2G_TRACE=gpurun_out/g3/trace_c4_$v.json timeout 300 python tools/trace_config.py c4 > gpurun_out/g3/trace_c4_$v.txt 2>&1
  python tools/trace_summary.py gpurun_out/g3/trace_c4_$v.json > gpurun_out/g3/trace_c4_${v}_summary.txt 2>&1
  rm -f gpurun_out/g3/trace_c4_$v.json
done
