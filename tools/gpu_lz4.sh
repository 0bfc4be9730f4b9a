#!/bin/bash
# LZ4 iteration: parity tests of every schedule, then the NP microbench (speculative kernel on, and off for reference)
TAG=${1:-lz4}; FILT=${2:-"hc=9"}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 -p no:cacheprovider -k "lz4" > gpurun_out/pytest_${TAG}.log 2>&1
echo "pytest rc=$?"; tail -4 gpurun_out/pytest_${TAG}.log
timeout 900 python tools/microbench.py NP --filter "$FILT" --steps 5 > gpurun_out/mb_${TAG}_spec.txt 2>&1; echo "mb rc=$?"
grep -h '^{' gpurun_out/mb_${TAG}_spec.txt | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print(d['case'], d['ms'], {k: v['ms'] for k, v in d['kernels'].items()})"
if [ -n "$NOSPEC" ]; then
CDM_LZ4_SPEC=0 timeout 900 python tools/microbench.py NP --filter "$FILT" --steps 5 > gpurun_out/mb_${TAG}_nospec.txt 2>&1; echo "mb0 rc=$?"
grep -h '^{' gpurun_out/mb_${TAG}_nospec.txt | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print('nospec', d['case'], d['ms'], {k: v['ms'] for k, v in d['kernels'].items()})"
fi
