cd $GRAFT_REPO_ROOT
bash tools/gpu_all.sh
bash tools/prof_launch.sh
K=${NCU_KERNEL:-k_topk_scan}
ncu --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 -o gpurun_out/full_$K -f python tools/c4_once.py C4 > gpurun_out/ncu_$K.log 2>&1; echo "ncu full $?"
