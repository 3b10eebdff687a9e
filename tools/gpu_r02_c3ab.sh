# c3 A/B on one box: previous builds vs the current one, and the current one with the new kernels off
O=gpurun_out/c3ab; mkdir -p $O; rm -f $O/*.txt
run() { python tools/run_config.py c3 0 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', d['ms_per_product'], d['ms_each'])" | tee -a $O/ab.txt; }
for i in 1 2; do
  H2G_LIB=build_ab/libh2g_old.so run old_a93e370
  H2G_LIB=build_ab/libh2g_old2.so run old_5936474
  run new
  H2G_GSUM_NO_LEAN=1 H2G_GSUM_NO_SUM=1 run new_no_lean_no_sum
  H2G_GSUM_NO_SUM=1 run new_no_sum
done
