#!/bin/bash
# bench value / e2e under stream-priority and FP-grid variants
for env in "CDM_RLE_PRIO=lo CDM_FP_GRID=p" "CDM_RLE_PRIO=hi CDM_FP_GRID=p" "CDM_RLE_PRIO=lo CDM_FP_GRID=t" "CDM_RLE_PRIO=hi CDM_FP_GRID=t"; do
  env $env timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('$env', 'value', d['value'], 'ms', d['ms_per_step'], 'fam', r['families_ms_per_step'], 'e2e', d['e2e']['value'])"
done
