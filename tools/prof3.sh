python tools/c4_once.py > gpurun_out/c4_once.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_tcf_scan -s 2 -c 1 -o gpurun_out/prof_tcf3 python tools/c4_once.py > gpurun_out/ncu3.log 2>&1; echo "ncu $?"
