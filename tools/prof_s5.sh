#!/bin/bash
# ncu --set full captures of the mid-size C4 MST kernels (second solve of tools/c4_once.py)
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out/s5
python tools/c4_once.py C4 > gpurun_out/s5/once.log 2>&1; echo "plain $?"
for k in k_cm_rowub k_cm_filter k_topk_scan k_tour1 k_cm_thresholds; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -o gpurun_out/s5/$k python tools/c4_once.py C4 > /dev/null 2>&1; echo "$k $?"
done
ncu --set full --clock-control none --import-source on -k regex:k_contract -s 3 -c 3 -o gpurun_out/s5/k_contract python tools/c4_once.py C4 > /dev/null 2>&1; echo "contract $?"
for f in gpurun_out/s5/*.ncu-rep; do python tools/ncu_summary.py $f; done > gpurun_out/s5/summary.txt 2>&1
