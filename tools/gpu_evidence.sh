#!/bin/bash
# one round of evidence: GPU tests, bench (config2), ncu launch list of the bench, ncu --set full of one batch
TAG=${1:-r01}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 -p no:cacheprovider > gpurun_out/pytest_${TAG}.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/pytest_${TAG}.log
timeout 600 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; echo "bench rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
   --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
echo "ncu launches rc=$?"
CDM_SERIAL=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fp_kernel|rle_kernel|rle_sums|scan_kernel|lz4_kernel" \
   -c 4 -o gpurun_out/prof_${TAG} -f python tools/one_batch.py 1 config2 > gpurun_out/ncu_full_${TAG}.log 2>&1
echo "ncu full rc=$?"
