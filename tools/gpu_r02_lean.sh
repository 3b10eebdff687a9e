# lean 2-factor gsum kernel: bitwise check against the 64x64 path, parity tests, c2/c4 A/B
mkdir -p gpurun_out/sum
for c in c2 c4; do
  H2G_GSUM_NO_SUM=1 H2G_GSUM_NO_LEAN=1 timeout 600 python tools/bitwise_z.py $c gpurun_out/sum/z_${c}_old.npz > /dev/null 2>&1
  timeout 600 python tools/bitwise_z.py $c gpurun_out/sum/z_${c}_new.npz > /dev/null 2>&1
  echo "$c: $(python tools/bitwise_z.py cmp gpurun_out/sum/z_${c}_old.npz gpurun_out/sum/z_${c}_new.npz 2>&1 | tail -3)" >> gpurun_out/sum/bitwise.txt
  rm -f gpurun_out/sum/z_${c}_*.npz
done
cat gpurun_out/sum/bitwise.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -3 > gpurun_out/sum/pytest.txt; cat gpurun_out/sum/pytest.txt
for i in 1 2; do
  for v in old new; do
    if [ $v = old ]; then export H2G_GSUM_NO_SUM=1; else unset H2G_GSUM_NO_SUM; fi
    for c in c4 c2; do
      python bench.py --config $c --steps 8 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v $c', round(d['ms_per_step'],2), round(d['e2e']['value']), round(d['roofline']['classes']['gsum']['ms'],1))" | tee -a gpurun_out/sum/ab.txt
    done
  done
done
