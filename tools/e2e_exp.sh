#!/bin/bash
for g in 1048576 2097152 4194304 16777216; do
  CDM_GROUP_MIN_BYTES=$g timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline > gpurun_out/e2e_$g.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/e2e_$g.json'));e=d['e2e'];print('group_min $g e2e',e['value'],'host_submit_ms',e['host_submit_ms_per_step'],'ms/step',round(144.06/e['value'],3))"
done
