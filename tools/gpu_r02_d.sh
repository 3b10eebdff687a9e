mkdir -p gpurun_out/g5
timeout 900 python -m pytest tests/test_gpu_stages.py -m gpu -q -x -rA > gpurun_out/g5/stages.txt 2>&1; echo "rc=$?" >> gpurun_out/g5/stages.txt
