#!/bin/bash
export H2G_SERIAL=1  # deterministic launch order so the list index matches the capture
# usage: tools/ncu_top.sh <kernel-regex> <out-name> [cmd...]
# Lists the kernel's launches (duration), then captures the longest one with --set full.
set -e
K=$1; OUT=$2; shift 2
ncu --kernel-name regex:$K --metrics gpu__time_duration.sum --clock-control none --csv "$@" > gpurun_out/${OUT}_list.csv 2>/dev/null
IDX=$(python - "$OUT" <<'PY'
import csv, sys
rows = [r for r in csv.reader(open(f"gpurun_out/{sys.argv[1]}_list.csv")) if len(r) > 10 and r[-3] == "gpu__time_duration.sum"]
mult = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "s": 1e6, "second": 1e6}
v = [float(r[-1].replace(",", "")) * mult.get(r[-2], 1.0) * 1e3 for r in rows]
i = max(range(len(v)), key=lambda k: v[k])
print(i)
print(f"{len(v)} launches, longest #{i} {v[i]/1e3:.1f} us, total {sum(v)/1e6:.2f} ms", file=sys.stderr)
PY
)
ncu --kernel-name regex:$K --launch-skip $IDX --launch-count 1 --set full --import-source on --clock-control none -o gpurun_out/$OUT -f "$@" > /dev/null 2>&1
