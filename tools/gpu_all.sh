cd $GRAFT_REPO_ROOT
export APPD_DEBUG_ROUNDS=1
python tools/c4_once.py C4 > gpurun_out/once.log 2>&1; echo "once $?"; grep -v "round [1-9]" gpurun_out/once.log | tail -4 | cut -c1-600
unset APPD_DEBUG_ROUNDS
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -15 gpurun_out/pytest_gpu.log
