O=gpurun_out/g52; mkdir -p $O
cap() {  # kernel regex, launch skip within the bench's profiled region, tag
  timeout 900 ncu --profile-from-start off --kernel-name-base demangled --kernel-name "regex:$1" --launch-skip $2 --launch-count 1 \
      --set full --import-source on --clock-control none -o $O/$3 -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/$3.log 2>&1
  ncu -i $O/$3.ncu-rep --page raw --csv > $O/$3_raw.csv 2> /dev/null
  python tools/ncu_stalls.py $O/$3.ncu-rep "$4" 40 > $O/$3_stalls.txt 2>&1
}
cap "gram_chol_kernel" 47 chol gram_chol
cap "svd_finish_kernel<16, 1>" 1 finish16 svd_finish
