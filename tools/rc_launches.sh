#!/bin/bash
# Launch list (gpu__time_duration) of one engine's sweeps through the constant-row path, summed per
# kernel, plus a --set full capture of one mid-sweep window launch (experiments; run under gpurun).
ENG=${1:-C4acamp}
python tools/time_c4.py $ENG > /dev/null
ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/rc_launches.csv python tools/time_c4.py $ENG > gpurun_out/rc_ncu_l.log 2>&1
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/rc_launches.csv')))
hi=next(i for i,r in enumerate(rows) if "Kernel Name" in r)
h=rows[hi]; ki,vi=h.index("Kernel Name"),h.index("Metric Value")
tot={};cnt={}
for r in rows[hi+1:]:
    if len(r)<=vi: continue
    k=r[ki][:90]; tot[k]=tot.get(k,0)+float(r[vi].replace(",","")); cnt[k]=cnt.get(k,0)+1
for k,v in sorted(tot.items(), key=lambda x:-x[1])[:12]:
    print(f"{v/1e6:10.3f} ms x{cnt[k]:5d}  {k}")
PY
