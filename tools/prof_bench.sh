# round-1 evidence: plain run, launch list, full captures of the two dominant kernels
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01_launches.csv $CMD > gpurun_out/r01_ncu_launch.log 2>&1; echo "launch list $?"
ncu --set full --clock-control none --import-source on -k regex:k_tcf_scan -s 6 -c 1 -o gpurun_out/r01_tcf_scan $CMD > gpurun_out/r01_ncu_tcf.log 2>&1; echo "tcf capture $?"
ncu --set full --clock-control none --import-source on -k 'regex:k_fill<' -s 1 -c 1 -o gpurun_out/r01_fill $CMD > gpurun_out/r01_ncu_fill.log 2>&1; echo "fill capture $?"
