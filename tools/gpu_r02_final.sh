# final evidence of the round: full GPU test suite, smoke, then tools/refresh_profiles.sh
mkdir -p gpurun_out/final
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/final/pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/final/pytest.txt
tail -3 gpurun_out/final/pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final/smoke.txt 2>&1; tail -1 gpurun_out/final/smoke.txt
ROUND=final bash tools/refresh_profiles.sh
