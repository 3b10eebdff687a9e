mkdir -p gpurun_out/g10
timeout 900 python -m pytest tests/test_gpu_shard.py -m gpu -q -x -rA > gpurun_out/g10/shard.txt 2>&1; echo "rc=$?" >> gpurun_out/g10/shard.txt
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/g10/tests.txt 2>&1; echo "rc=$?" >> gpurun_out/g10/tests.txt
