#!/bin/bash
# Round-2 evidence on one GPU: per-config times, the C4 bench line, its launch list, and
# ncu --set full captures of the dominant kernels (each after its command exited 0 without ncu).
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out/r02
python tools/cfg_times.py > gpurun_out/r02/cfg_times.log 2>&1; echo "cfg_times $?"
cp gpurun_out/cfg_times.txt gpurun_out/r02/ 2>/dev/null
python bench.py --steps 10 --warmup 3 > gpurun_out/r02/bench_c4.log 2>&1; echo "bench $?"; tail -1 gpurun_out/r02/bench_c4.log > gpurun_out/r02/bench_c4.json
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/r02/plain.log 2>&1; echo "plain $?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02/launches_c4_bench.csv $CMD > /dev/null 2>&1; echo "launch list $?"
python tools/launches.py gpurun_out/r02/launches_c4_bench.csv > gpurun_out/r02/launches_summary.txt
ncu --set full --clock-control none --import-source on -k regex:^k_fill$ -s 1 -c 1 -o gpurun_out/r02/full_fill $CMD > /dev/null 2>&1; echo "fill $?"
ncu --set full --clock-control none --import-source on -k regex:k_tcf_scan -s 2 -c 2 -o gpurun_out/r02/full_tcf $CMD > /dev/null 2>&1; echo "tcf $?"
ncu --set full --clock-control none --import-source on -k regex:k_list_exact -s 2 -c 2 -o gpurun_out/r02/full_list $CMD > /dev/null 2>&1; echo "list $?"
ncu --set full --clock-control none --import-source on -k regex:k_topk_scan -s 1 -c 1 -o gpurun_out/r02/full_topk $CMD > /dev/null 2>&1; echo "topk $?"
ncu --set full --clock-control none --import-source on -k regex:"k_tc_prep|k_list_sort" -s 3 -c 3 -o gpurun_out/r02/full_prep $CMD > /dev/null 2>&1; echo "prep $?"
python tools/cfg_times.py C1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_prim -s 3 -c 2 -o gpurun_out/r02/full_prim python tools/cfg_times.py C1 > /dev/null 2>&1; echo "prim $?"
ncu --set full --clock-control none --import-source on -k regex:"k_validate_square|k_scan_weights_topk|k_fill" -s 6 -c 3 -o gpurun_out/r02/full_c3 python tools/cfg_times.py C3 > /dev/null 2>&1; echo "c3 $?"
for r in fill tcf list topk prep prim c3; do python tools/ncu_summary.py gpurun_out/r02/full_$r.ncu-rep > gpurun_out/r02/r02_$r.metrics.txt 2>&1; done
ls -la gpurun_out/r02
# late round 2: the cooperative kernels on the lighter grid barrier (tours, contraction)
ncu --set full --clock-control none --import-source on -k regex:"k_tour1|k_tour2|k_contract" -s 3 -c 3 -o gpurun_out/r02/full_coop $CMD > /dev/null 2>&1; echo "coop $?"
python tools/ncu_summary.py gpurun_out/r02/full_coop.ncu-rep > gpurun_out/r02/r02_coop.metrics.txt 2>&1
# (the GPU suite runs separately)
rm -f gpurun_out/r02/*.ncu-rep; du -sh gpurun_out
