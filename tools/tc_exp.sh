cd $GRAFT_REPO_ROOT
for e in 0 3 4 5 6; do
  APPD_TC_EXPERIMENT=$e python tools/c4_once.py C4 0 -1 > gpurun_out/exp_$e.log 2>&1
  echo "exp $e: $(tail -1 gpurun_out/exp_$e.log | python -c "import sys,ast; d=ast.literal_eval(sys.stdin.read()); print('tcscan', round(d['ms_tcscan'],3), 'launches', d['tcscan_launches'], 'mst', round(d['ms_mst'],3))")"
done
