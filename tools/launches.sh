#!/bin/bash
# per-kernel device times for one workload (serial families), summarised
WL=${1:-config2}
CDM_SERIAL=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_$WL.csv python tools/one_batch.py 2 $WL > /dev/null 2>&1
python - <<PY
import csv, collections
rows=[r for r in csv.reader(open('gpurun_out/launches_$WL.csv')) if len(r)>5]
h=rows[0]; k=h.index('Kernel Name'); v=h.index('Metric Value'); g=h.index('Grid Size')
agg=collections.defaultdict(list)
for r in rows[1:]: agg[(r[k][:48], r[g])].append(float(r[v].replace(',',''))/1e3)
for key,vals in agg.items(): print(f"$WL {key[0]:48s} {key[1]:16s} n={len(vals)} mean={sum(vals)/len(vals):9.2f} us")
PY
