cd $GRAFT_REPO_ROOT
for s in 0 10 20; do
APPD_TC_BENCH=1 ncu --set full --clock-control none -k regex:k_tcf_scan -s $s -c 1 -o gpurun_out/tcexp_$s python tools/c4_once.py C4 > gpurun_out/tcexp_$s.log 2>&1; echo "cap $s $?"
done
