O=gpurun_out/g55; mkdir -p $O
for i in 1 2; do
timeout 300 python tools/run_config.py c4 0 5 > $O/c4_$i.json 2>&1
H2G_GRAM_PROT=1 timeout 300 python tools/run_config.py c4 0 5 > $O/c4_prot_$i.json 2>&1
done
H2G_GRAM_PROT=1 timeout 300 python tools/run_config.py c2 0 5 > $O/c2_prot.json 2>&1
timeout 300 python tools/run_config.py c2 0 5 > $O/c2.json 2>&1
