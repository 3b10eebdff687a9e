mkdir -p gpurun_out/g1
nvidia-smi --query-gpu=name,clocks.sm --format=csv > gpurun_out/g1/smi.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/g1/pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/g1/pytest.txt
for c in c2 c4; do
H2G_TRACE=gpurun_out/g1/trace_$c.json timeout 300 python tools/trace_config.py $c > gpurun_out/g1/trace_$c.txt 2>&1
python tools/trace_summary.py gpurun_out/g1/trace_$c.json > gpurun_out/g1/trace_${c}_summary.txt 2>&1
done
H2G_DEBUG_SWEEPS=1 timeout 300 python tools/trace_config.py c4 > gpurun_out/g1/sweeps_c4.txt 2>&1
timeout 300 python tools/run_config.py c4 > gpurun_out/g1/full_c4.json 2>&1
