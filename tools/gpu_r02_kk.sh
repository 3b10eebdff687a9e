O=gpurun_out/g65; mkdir -p $O
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/run_config.py c5 65536 1 > $O/launches_c5.csv 2> /dev/null
python tools/launch_summary.py $O/launches_c5.csv 30 > $O/launches_c5_summary.txt 2>&1
H2G_DEBUG_SWEEPS=1 H2G_SERIAL=1 timeout 600 python tools/run_config.py c5 65536 1 > $O/sweeps_c5.txt 2>&1
