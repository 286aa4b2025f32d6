cd $GRAFT_REPO_ROOT
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python tools/cfg_times.py C3 > gpurun_out/ncu_c3.log 2>&1; echo "ncu $?"
python - <<'PY'
import csv, collections
rows=list(csv.reader(open('gpurun_out/launches_c3.csv')))
hi=next(i for i,r in enumerate(rows) if 'Kernel Name' in r); hdr=rows[hi]; data=rows[hi+1:]
ki=hdr.index('Kernel Name'); vi=hdr.index('Metric Value')
data=data[2*len(data)//3:]
agg=collections.OrderedDict()
for r in data:
    nm=r[ki].split('(')[0][:50]; a=agg.setdefault(nm,[0,0.0]); a[0]+=1; a[1]+=float(r[vi].replace(',',''))
for k,(c,t) in sorted(agg.items(), key=lambda x:-x[1][1])[:12]: print(f"{k:50s} {c:4d} {t/1e3:9.1f} us")
PY
