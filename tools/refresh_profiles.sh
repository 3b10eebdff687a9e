#!/bin/bash
# Regenerate the round's evidence on the GPU box (run from the repo root, under gpurun): the driver's
# default bench line (c4), the ncu launch list of its timed region (cudaProfilerStart/Stop: every
# engine thread and stream), ncu --set full captures of the dominant kernel's largest launches, a
# like-for-like c2 pair at n = 16,384 (GPU bench and the CPU reference arm at the same n), and the
# full-size runs.  Outputs land in gpurun_out/$R/; copy what is judged into profiles/.
set -u
R=${ROUND:-r02}
O=gpurun_out/$R
mkdir -p $O
python bench.py --steps 10 --warmup 3 > $O/bench_c4.json 2> $O/bench_c4.err; echo "bench c4 rc=$?"
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/launches_c4.csv 2> /dev/null; echo "launch list rc=$?"
python tools/launch_summary.py $O/launches_c4.csv 40 > $O/launches_c4_summary.txt
cap() {  # kernel regex, launch skip (within tools/run_config.py c4 0 1), tag
  ncu --kernel-name-base demangled --kernel-name "regex:$1" --launch-skip $2 --launch-count 1 --set full --import-source on \
      --clock-control none -o $O/$3 -f python tools/run_config.py c4 0 1 > $O/$3.log 2>&1
  ncu -i $O/$3.ncu-rep --page raw --csv > $O/$3_raw.csv 2> /dev/null
  python tools/ncu_stalls.py $O/$3.ncu-rep "$4" 30 > $O/$3_stalls.txt 2>&1
}
cap "gsum_pipe_kernel<.int.1>" 0 gsum_dense gsum_pipe
cap "gram_dd_partial_kernel" 60 gram gram_dd
bash tools/gpu_r02_lean2.sh > /dev/null 2>&1; cp gpurun_out/lean2/lean_stalls.txt $O/lean_stalls.txt  # longest gsum_lean_kernel launch of a serialized product
python bench.py --config c2 --steps 10 --warmup 3 > $O/bench_c2.json 2> $O/bench_c2.err; echo "bench c2 rc=$?"
python bench.py --impl reference --config c2 --cpu-sample-n 16384 --steps 1 --warmup 0 > $O/ref_c2_16384.json 2> $O/ref_c2.err; echo "ref c2 rc=$?"
for c in c2 c3 c4; do python tools/run_config.py $c 0 5 > $O/full_$c.json 2> $O/full_$c.err; done
H2G_TRACE=$O/trace_c4.json python tools/trace_config.py c4 > /dev/null 2>&1
python tools/trace_summary.py $O/trace_c4.json > $O/trace_c4_summary.txt; rm -f $O/trace_c4.json
echo done
