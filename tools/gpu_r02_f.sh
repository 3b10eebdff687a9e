mkdir -p gpurun_out/g7
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_stages.py -m gpu -q -x > gpurun_out/g7/tests.txt 2>&1; echo "rc=$?" >> gpurun_out/g7/tests.txt
timeout 300 python tools/run_config.py c4 0 3 > gpurun_out/g7/c4.json 2>&1
timeout 300 python tools/run_config.py c2 0 5 > gpurun_out/g7/c2.json 2>&1
H2G_NO_DEFER_OUT=1 timeout 300 python tools/run_config.py c4 0 3 > gpurun_out/g7/c4_nodefer.json 2>&1
cap() {  # name regex, skip, tag
  timeout 600 ncu --kernel-name-base demangled --kernel-name "regex:$1" --launch-skip $2 --launch-count 1 --set full --import-source on \
    --clock-control none -o gpurun_out/g7/$3 -f python tools/run_config.py c4 0 1 > gpurun_out/g7/$3.log 2>&1
  ncu -i gpurun_out/g7/$3.ncu-rep --page raw --csv > gpurun_out/g7/$3_raw.csv 2>/dev/null
  python tools/ncu_stalls.py gpurun_out/g7/$3.ncu-rep "$4" 30 > gpurun_out/g7/$3_stalls.txt 2>&1
}
cap "gsum_pipe_kernel<.int.1>" 0 gsum1 gsum_pipe
cap "gsum_pipe_kernel<.int.0>" 140 gsum0_a gsum_pipe
cap "gram_dd_partial_kernel" 70 gram gram_dd
cap "svd_finish_kernel<.int.24, .bool.1>" 0 svdfin24 svd_finish
