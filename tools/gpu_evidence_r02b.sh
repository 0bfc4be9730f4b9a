#!/bin/bash
# round-2 closing evidence: headline + the other workloads' bench lines with the current kernels / schedule
TAG=${1:-r02m}
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_${TAG}_config4.json 2> gpurun_out/bench_${TAG}_config4.err; echo "config4 rc=$?"
timeout 900 python bench.py --workload config4sd --no-cpu-baseline > gpurun_out/bench_${TAG}_config4sd.json 2>/dev/null; echo "config4sd rc=$?"
timeout 900 python bench.py --workload partsupp --no-cpu-baseline > gpurun_out/bench_${TAG}_partsupp.json 2>/dev/null; echo "partsupp rc=$?"
timeout 1500 python bench.py --workload config5 --no-cpu-baseline > gpurun_out/bench_${TAG}_config5.json 2>gpurun_out/bench_${TAG}_config5.err; echo "config5 rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_${TAG}_reference.json 2>/dev/null; echo "reference rc=$?"
