O=gpurun_out/g70; mkdir -p $O
timeout 300 python tools/sanitize_case.py rand_s2_2d > $O/plain.txt 2>&1 && \
timeout 900 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 7 python tools/sanitize_case.py rand_s2_2d > $O/memcheck.txt 2>&1; echo "rc=$?" >> $O/memcheck.txt
