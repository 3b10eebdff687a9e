# re-entry check: GPU tests, smoke, default bench line, reference arm
mkdir -p gpurun_out/re1
nvidia-smi --query-gpu=name,clocks.sm --format=csv > gpurun_out/re1/smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/re1/pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/re1/pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/re1/smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/re1/bench.txt 2>&1; echo "bench rc=$?" >> gpurun_out/re1/bench.txt
tail -3 gpurun_out/re1/pytest.txt; tail -2 gpurun_out/re1/smoke.txt; tail -2 gpurun_out/re1/bench.txt
