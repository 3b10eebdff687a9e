#!/bin/bash
# Regenerate the round's evidence on the GPU box (run from the repo root, under gpurun):
#   bench line, ncu launch list of the timed region, one ncu --set full capture of the dominant
#   kernel's longest launch, trace summary, full-size c3 / c4 runs.  Outputs land in gpurun_out/;
#   copy what is to be judged into profiles/ (tools/refresh_profiles.sh is the recipe).
set -u
R=${ROUND:-r01}
mkdir -p gpurun_out
python bench.py --steps 10 --warmup 3 > gpurun_out/${R}_bench_c2.json 2> gpurun_out/${R}_bench_c2.err
echo "bench rc=$?"
# launch list of the timed region only (NVTX range "timed"), cold-cache serialised per-launch times
ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${R}_launches_c2.csv 2> /dev/null
echo "launch list rc=$?"
python tools/launch_summary.py gpurun_out/${R}_launches_c2.csv > gpurun_out/${R}_launches_c2_summary.txt
# the dense-target assembly launch (gsum_mma_kernel<1>, the longest GEMM launch of a product)
ncu --kernel-name-base demangled --kernel-name regex:"gsum_mma_kernel<.int.1>" --launch-skip 3 --launch-count 1 --set full --import-source on \
    --clock-control none -o gpurun_out/${R}_gsum -f python tools/trace_config.py c2 > /dev/null 2>&1
echo "gsum capture rc=$?"
ncu -i gpurun_out/${R}_gsum.ncu-rep --page raw --csv > gpurun_out/${R}_gsum_raw.csv 2> /dev/null
python tools/ncu_stalls.py gpurun_out/${R}_gsum.ncu-rep gsum_mma 30 > gpurun_out/${R}_gsum_stalls.txt 2> /dev/null
H2G_TRACE=gpurun_out/${R}_trace_c2.json python tools/trace_config.py c2 > /dev/null 2>&1
python tools/trace_summary.py gpurun_out/${R}_trace_c2.json > gpurun_out/${R}_trace_c2_summary.txt
for c in c3 c4; do python tools/run_config.py $c > gpurun_out/${R}_full_$c.json 2> gpurun_out/${R}_full_$c.err; done
echo done
