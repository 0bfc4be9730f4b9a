#!/bin/bash
# bench + ncu evidence for one round (tag = $1, e.g. r01)
TAG=${1:-r01}
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; echo "bench rc=$?"
cat gpurun_out/bench_${TAG}.json
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_${TAG}.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
   --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 3 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fp_kernel|rle_kernel|inner_kernel|scan_kernel" \
   -s 8 -c 8 -o gpurun_out/prof_${TAG} -f python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_full_${TAG}.log 2>&1
echo "ncu full rc=$?"
