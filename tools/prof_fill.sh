cd $GRAFT_REPO_ROOT
CMD="python tools/c4_once.py C4"
ncu --set full --clock-control none --import-source on -k regex:^k_fill$ -s 1 -c 1 -o gpurun_out/full_fill $CMD > gpurun_out/ncu_fill.log 2>&1; echo "fill capture $?"; tail -3 gpurun_out/ncu_fill.log
