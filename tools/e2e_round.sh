#!/bin/bash
# e2e experiments: pytest gpu, bench line, timelines
mkdir -p gpurun_out
TAG=${1:-e2e}
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 -p no:cacheprovider > gpurun_out/pytest_${TAG}.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/pytest_${TAG}.log
timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/bench_${TAG}.json 2>gpurun_out/bench_${TAG}.err
python -c "
import json; d=json.load(open('gpurun_out/bench_${TAG}.json'))
print('value', d['value'], 'ms', d['ms_per_step'], 'fam', d['roofline']['families_ms_per_step'], 'e2e', d['e2e'])"
tail -3 gpurun_out/bench_${TAG}.err
timeout 300 python tools/e2e_timeline.py config2 pipeline > gpurun_out/e2e_tl_${TAG}.txt 2>&1; head -3 gpurun_out/e2e_tl_${TAG}.txt
cp gpurun_out/e2e_trace_config2.json gpurun_out/e2e_trace_pipe.json
timeout 300 python tools/e2e_timeline.py config2 submit > gpurun_out/e2e_tl_sub_${TAG}.txt 2>&1; head -3 gpurun_out/e2e_tl_sub_${TAG}.txt
