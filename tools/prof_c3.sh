cd $GRAFT_REPO_ROOT
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python tools/c4_once.py C3 > gpurun_out/ncu_c3.log 2>&1; echo "ncu $?"
python tools/launches.py gpurun_out/launches_c3.csv | head -8
ncu --set full --clock-control none --import-source on -k regex:k_scan_weights_topk -s 1 -c 1 -o gpurun_out/full_wtopk -f python tools/c4_once.py C3 > gpurun_out/ncu_wtopk.log 2>&1; echo "ncu wtopk $?"
