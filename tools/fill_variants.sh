cd $GRAFT_REPO_ROOT
for r in 1 2 3; do
  python tools/c4_once.py C4 > gpurun_out/fv.log 2>&1
  echo "run $r: $(tail -1 gpurun_out/fv.log | grep -o "'ms_fill': [0-9.]*") $(tail -1 gpurun_out/fv.log | grep -o "'ms_total': [0-9.]*")"
done
