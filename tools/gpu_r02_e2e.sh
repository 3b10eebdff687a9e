# deferred nearfield upload: parity tests (incl. first-use paths), then the c4 bench line twice (e2e seconds)
O=gpurun_out/e2e; mkdir -p $O; rm -f $O/*.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -3 | tee $O/pytest.txt
for i in 1 2 3; do
  python bench.py --config c4 --steps 8 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c4', round(d['ms_per_step'],2), round(d['e2e']['value']), round(d['e2e']['seconds']*1e3,1))" | tee -a $O/ab.txt
done
timeout 300 python tools/e2e_split_c4.py 2>&1 | tail -7 | tee $O/split.txt
