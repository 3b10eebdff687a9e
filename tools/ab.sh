#!/bin/bash
# A/B timing of two builds of libh2g.so in one box session:
#   tools/ab.sh <lib_a> <lib_b> [rounds] [bench args...]
# alternates bench.py runs (device ms/step, e2e DOF/s) between the two libraries.
A=$1; B=$2; R=${3:-3}; shift 3
for i in $(seq $R); do
  for L in $A $B; do
    H2G_LIB=$L python bench.py --steps 10 --warmup 3 --no-cpu-baseline "$@" 2>/dev/null | \
      python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$L', round(d['ms_per_step'],2), round(d['e2e']['value']))"
  done
done
