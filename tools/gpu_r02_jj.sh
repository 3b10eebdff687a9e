O=gpurun_out/g64; mkdir -p $O
for c in c2 c3 c4; do timeout 300 python tools/run_config.py $c 0 5 > $O/full_$c.json 2> $O/full_$c.err; done
timeout 600 python tools/run_config.py c5 65536 5 > $O/full_c5_65536.json 2> $O/full_c5.err
timeout 900 python -m pytest tests/test_gpu_shard.py -m gpu -q -s > $O/shard.txt 2>&1; echo "rc=$?" >> $O/shard.txt
