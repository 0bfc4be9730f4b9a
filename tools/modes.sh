#!/bin/bash
# compare concurrent vs serial kernel families (bench + trace)
for mode in concurrent serial; do
  if [ $mode == serial ]; then export CDM_SERIAL=1; fi
  echo "=== $mode"
  timeout 300 python bench.py --no-cpu-baseline --steps 100 > gpurun_out/bench_$mode.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/bench_$mode.json'));print('value',d['value'],'e2e',d['e2e']['value'],'fam',d['roofline']['families_ms_per_step'])"
  timeout 300 python tools/trace_rle.py
done
