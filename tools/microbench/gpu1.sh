set -x
nproc; lscpu | grep -E "Model name|Socket|Core|Thread"; free -g; nvidia-smi; df -h /tmp | tail -1
./tools/microbench/mb > gpurun_out/mb.log 2>&1; echo "exit $?"; cat gpurun_out/mb.log
