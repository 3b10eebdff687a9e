# ncu: launch list of the lean gsum kernel in the bench's profiled step + full capture of its longest launch
O=gpurun_out/lean2; mkdir -p $O
export H2G_SERIAL=1
timeout 900 ncu --profile-from-start off --kernel-name-base demangled --kernel-name "regex:gsum_lean" --metrics gpu__time_duration.sum --clock-control none --csv \
   python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/lean_list.csv 2> /dev/null
IDX=$(python - <<'PY'
import csv
rows = [r for r in csv.reader(open("gpurun_out/lean2/lean_list.csv")) if len(r) > 10 and r[-3] == "gpu__time_duration.sum"]
v = [float(r[-1].replace(",", "")) for r in rows]
i = max(range(len(v)), key=lambda k: v[k])
print(i)
PY
)
echo "longest lean launch index $IDX" > $O/info.txt
timeout 900 ncu --profile-from-start off --kernel-name-base demangled --kernel-name "regex:gsum_lean" --launch-skip $IDX --launch-count 1 \
   --set full --import-source on --clock-control none -o $O/lean -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/lean.log 2>&1
ncu -i $O/lean.ncu-rep --page raw --csv > $O/lean_raw.csv 2> /dev/null
python tools/ncu_stalls.py $O/lean.ncu-rep gsum_lean 40 > $O/lean_stalls.txt 2>&1
head -3 $O/lean_stalls.txt | cut -c1-400
