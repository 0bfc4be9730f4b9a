#!/bin/bash
# one GPU call: smoke + pytest -m gpu + default bench line (each bounded by timeout)
TAG=${1:-r02f}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu_${TAG}.txt 2>&1
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke_${TAG}.log 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider ${KEXPR:+-k "$KEXPR"} > gpurun_out/pytest_${TAG}.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_${TAG}.log
if [ -z "$NO_BENCH" ]; then
timeout 900 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; echo "bench rc=$?"
fi
