cd $GRAFT_REPO_ROOT
python tools/c4_once.py C4 > gpurun_out/once.log 2>&1; echo "plain $?"; tail -1 gpurun_out/once.log | cut -c1-400
for K in k_chunk_exact k_cm_exact k_topk_thr k_topk_select k_cm_filter; do
ncu --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 -o gpurun_out/full_$K python tools/c4_once.py C4 > gpurun_out/ncu_$K.log 2>&1; echo "$K $?"
done
