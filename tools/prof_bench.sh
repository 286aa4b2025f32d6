# tests + bench line + launch list + full captures of the dominant kernels (one GPU)
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/pytest_gpu.log
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_full.log 2>&1; echo "bench $?"; tail -1 gpurun_out/bench_full.log | cut -c1-200
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/prof_plain.log 2>&1; echo "plain $?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "launch list $?"
python tools/launches.py gpurun_out/launches.csv > gpurun_out/launches_summary.txt; head -24 gpurun_out/launches_summary.txt
ncu --set full --clock-control none --import-source on -k regex:^k_fill$ -s 1 -c 1 -o gpurun_out/full_fill $CMD > gpurun_out/ncu_fill.log 2>&1; echo "fill capture $?"
ncu --set full --clock-control none --import-source on -k regex:k_tcf_scan -s 2 -c 2 -o gpurun_out/full_tcf $CMD > gpurun_out/ncu_tcf.log 2>&1; echo "tcf capture $?"
ncu --set full --clock-control none --import-source on -k regex:k_list_exact -s 2 -c 2 -o gpurun_out/full_list $CMD > gpurun_out/ncu_list.log 2>&1; echo "list capture $?"
ncu --set full --clock-control none --import-source on -k regex:k_topk_scan -s 1 -c 1 -o gpurun_out/full_topk $CMD > gpurun_out/ncu_topk.log 2>&1; echo "topk capture $?"
