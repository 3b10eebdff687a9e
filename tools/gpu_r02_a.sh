mkdir -p gpurun_out/g2
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -x -rA > gpurun_out/g2/fullsize.txt 2>&1; echo "rc=$?" >> gpurun_out/g2/fullsize.txt
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/g2/bench.json 2> gpurun_out/g2/bench.err; echo "rc=$?" >> gpurun_out/g2/bench.err
