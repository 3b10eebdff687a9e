O=gpurun_out/g68; mkdir -p $O
cap() {
  timeout 900 ncu --profile-from-start off --kernel-name-base demangled --kernel-name "regex:$1" --launch-skip $2 --launch-count 1 \
      --set full --import-source on --clock-control none -o $O/$3 -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/$3.log 2>&1
  ncu -i $O/$3.ncu-rep --page raw --csv > $O/$3_raw.csv 2> /dev/null
  python tools/ncu_stalls.py $O/$3.ncu-rep "$4" 30 > $O/$3_stalls.txt 2>&1
}
cap "svd_finish_kernel<.int.16, .bool.1>" 1 finish16 svd_finish
cap "tile_absorb_kernel" 2 tile tile_absorb
cap "gsum_whole_kernel" 0 whole gsum_whole
