cd $GRAFT_REPO_ROOT
bash tools/gpu_all.sh
bash tools/prof_launch.sh
python tools/cfg_times.py > gpurun_out/cfg_times.log 2>&1; tail -8 gpurun_out/cfg_times.log
