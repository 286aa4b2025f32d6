cd $GRAFT_REPO_ROOT
python tools/c4_once.py C4 > gpurun_out/once.log 2>&1; echo "plain $?"; tail -2 gpurun_out/once.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cache.csv python tools/c4_once.py C4 > gpurun_out/ncu_once.log 2>&1; echo "ncu $?"
python tools/launches.py gpurun_out/launches_cache.csv > gpurun_out/launches_cache_summary.txt 2>&1; cat gpurun_out/launches_cache_summary.txt | head -40
