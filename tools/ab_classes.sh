#!/bin/bash
# kernel-class device ms (profile mode) of two library builds, alternating: tools/ab_classes.sh A B [rounds]
A=$1; B=$2; R=${3:-2}
for i in $(seq $R); do
  for L in $A $B; do
    H2G_LIB=$L python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | \
      python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); c=d['roofline']['classes']; print('$L', round(d['ms_per_step'],2), {k: round(v['ms'],2) for k,v in c.items() if v['ms']>0})"
  done
done
