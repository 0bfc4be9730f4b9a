#!/bin/bash
for sub in 16384 65536; do for g in 0 1; do
  if [ $g == 1 ]; then export CDM_LZ4_GLOBAL=1; else unset CDM_LZ4_GLOBAL; fi
  CDM_SERIAL=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:lz4 \
    --log-file gpurun_out/lz4_${sub}_${g}.csv python tools/one_batch.py 1 config3 $sub > /dev/null 2>&1
  python -c "
import csv
rows=[r for r in csv.reader(open('gpurun_out/lz4_${sub}_${g}.csv')) if len(r)>5]
h=rows[0]; v=h.index('Metric Value'); k=h.index('Kernel Name')
print('sub=$sub global=$g', [ (r[k][15:30], float(r[v].replace(',',''))/1e3) for r in rows[1:]])
"
done; done
