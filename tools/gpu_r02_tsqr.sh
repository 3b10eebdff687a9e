# ncu --set full of the longest svd_tsqr_kernel and tile_absorb_kernel launches of a serialized c4 product
O=gpurun_out/tsqr; mkdir -p $O
export H2G_SERIAL=1
cap() {
  timeout 900 ncu --profile-from-start off --kernel-name-base demangled --kernel-name "regex:$1" --metrics gpu__time_duration.sum --clock-control none --csv \
     python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/$2_list.csv 2> /dev/null
  IDX=$(python - $O/$2_list.csv <<'PY'
import csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10 and r[-3] == "gpu__time_duration.sum"]
v = [float(r[-1].replace(",", "")) for r in rows]
print(max(range(len(v)), key=lambda k: v[k]))
PY
)
  timeout 900 ncu --profile-from-start off --kernel-name-base demangled --kernel-name "regex:$1" --launch-skip $IDX --launch-count 1 \
     --set full --import-source on --clock-control none -o $O/$2 -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/$2.log 2>&1
  ncu -i $O/$2.ncu-rep --page raw --csv > $O/$2_raw.csv 2> /dev/null
  python tools/ncu_stalls.py $O/$2.ncu-rep "$1" 40 > $O/$2_stalls.txt 2>&1
  rm -f $O/$2.ncu-rep
  head -2 $O/$2_stalls.txt | cut -c1-300
}
cap svd_tsqr_kernel tsqr
