# quick check of a kernel change: bitwise Z against the 64x64 tile path at c2/c4, c4 bench twice
O=gpurun_out/quick; mkdir -p $O; rm -f $O/*.txt
for c in c2 c4; do
  H2G_GSUM_NO_SUM=1 H2G_GSUM_NO_LEAN=1 timeout 600 python tools/bitwise_z.py $c $O/z_${c}_old.npz > /dev/null 2>&1
  timeout 600 python tools/bitwise_z.py $c $O/z_${c}_new.npz > /dev/null 2>&1
  echo "$c: $(python tools/bitwise_z.py cmp $O/z_${c}_old.npz $O/z_${c}_new.npz 2>&1 | tail -3)" | tee -a $O/bitwise.txt
  rm -f $O/z_${c}_*.npz
done
for i in 1 2; do
  for c in c4 c2; do
    python bench.py --config $c --steps 8 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c', round(d['ms_per_step'],2), round(d['e2e']['value']), round(d['roofline']['classes']['gsum']['ms'],1))" | tee -a $O/ab.txt
  done
done
