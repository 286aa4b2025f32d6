for e in 0 3 5 6; do
  APPD_TC_EXPERIMENT=$e timeout 120 python tools/c4_exp.py > gpurun_out/exp_$e.log 2>&1
  APPD_TC_EXPERIMENT=$e ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_tcf_scan -c 3 --csv --log-file gpurun_out/exp_$e.csv python tools/c4_exp.py > /dev/null 2>&1
  echo "exp $e: $(grep k_tcf_scan gpurun_out/exp_$e.csv | awk -F'","' '{print $NF}' | tr -d '"' | tr '\n' ' ')"
done
