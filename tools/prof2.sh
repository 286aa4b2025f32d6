python tools/c4_once.py > gpurun_out/c4_once.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r2.csv python tools/c4_once.py > gpurun_out/ncu1.log 2>&1; echo "ncu1 $?"
ncu --set full --clock-control none --import-source on -k regex:k_tcf_scan -s 2 -c 1 -o gpurun_out/prof_tcf2 python tools/c4_once.py > gpurun_out/ncu2.log 2>&1; echo "ncu2 $?"
