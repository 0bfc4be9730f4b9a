#!/bin/bash
mkdir -p gpurun_out
for conn in 8 32; do
  CUDA_DEVICE_MAX_CONNECTIONS=$conn timeout 300 python tools/graph_lag.py 2>/dev/null | tail -7 | sed "s/^/conn$conn /"
  CUDA_DEVICE_MAX_CONNECTIONS=$conn timeout 300 python tools/e2e_timeline.py config2 pipeline > /dev/null 2>&1
  cp gpurun_out/e2e_trace_config2.json gpurun_out/e2e_trace_c$conn.json
  CUDA_DEVICE_MAX_CONNECTIONS=$conn timeout 300 python bench.py --steps 80 --warmup 5 --no-cpu-baseline > gpurun_out/b_c$conn.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/b_c$conn.json'));print('conn $conn e2e',d['e2e']['value'], 'submit', d['e2e']['submit_batch']['value'], 'value', d['value'])"
done
