#!/bin/bash
# ANS A/B: the ANS GPU parity tests, then --workload ans / strdict bench lines (value, ans kernel ms), twice
timeout 600 python -m pytest tests -m gpu -q -x -k "ans or strdict" -p no:cacheprovider 2>&1 | tail -1
for rep in 1 2; do
  for w in ans strdict; do
    r=$(timeout 300 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print(d['value'], d['roofline']['kernels_ms_per_step'].get('ans_warp_kernel'))")
    echo "$w $r"
  done
done
