#!/bin/bash
# trimmed round-end evidence: GPU tests, headline + reference + ans + strdict bench lines, launch list, ncu full of the ANS/StrDict kernels
TAG=${1:-r01h}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 -p no:cacheprovider > gpurun_out/pytest_${TAG}.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/pytest_${TAG}.log
timeout 600 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; echo "bench rc=$?"
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_${TAG}.json 2>&1
timeout 600 python bench.py --workload ans --steps 20 --warmup 3 > gpurun_out/bench_ans_${TAG}.json 2>/dev/null
timeout 600 python bench.py --workload strdict --steps 10 --warmup 3 > gpurun_out/bench_strdict_${TAG}.json 2>/dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
   --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
echo "ncu launches rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
   --log-file gpurun_out/launches_ans_${TAG}.csv python bench.py --workload ans --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
echo "ncu ans launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sd_|ans_" \
   -c 4 -o gpurun_out/prof_ans_${TAG} -f python tools/one_batch.py 1 ans > gpurun_out/ncu_ans_${TAG}.log 2>&1
echo "ncu ans full rc=$?"
