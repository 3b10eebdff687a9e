O=gpurun_out/g69; mkdir -p $O
for i in 1 2; do
timeout 300 python tools/run_config.py c4 0 5 > $O/c4_$i.json 2>&1
H2G_GSUM_NO_WHOLE=1 timeout 300 python tools/run_config.py c4 0 5 > $O/c4_nowhole_$i.json 2>&1
done
