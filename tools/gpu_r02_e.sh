mkdir -p gpurun_out/g6
cap() {  # name regex, skip, tag
  timeout 600 ncu --kernel-name-base demangled --kernel-name "regex:$1" --launch-skip $2 --launch-count 1 --set full --import-source on \
    --clock-control none -o gpurun_out/g6/$3 -f python tools/run_config.py c4 0 1 > gpurun_out/g6/$3.log 2>&1
  ncu -i gpurun_out/g6/$3.ncu-rep --page raw --csv > gpurun_out/g6/$3_raw.csv 2>/dev/null
  python tools/ncu_stalls.py gpurun_out/g6/$3.ncu-rep "$4" 30 > gpurun_out/g6/$3_stalls.txt 2>&1
}
cap "gsum_pipe_kernel<1>" 0 gsum1 gsum_pipe
cap "gsum_pipe_kernel<0>" 105 gsum0_push gsum_pipe
cap "gram_dd_partial_kernel" 47 gram gram_dd
cap "svd_finish_kernel<24, 1>" 0 svdfin24 svd_finish
