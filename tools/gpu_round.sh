#!/bin/bash
# tests + bench (+ optional ncu) in one GPU call.  usage: gpu_round.sh TAG [ncu]
TAG=${1:-dev}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 -p no:cacheprovider ${PYTEST_ARGS} > gpurun_out/pytest_${TAG}.log 2>&1
echo "pytest rc=$?"; tail -15 gpurun_out/pytest_${TAG}.log
timeout 600 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; echo "bench rc=$?"
cat gpurun_out/bench_${TAG}.json; tail -3 gpurun_out/bench_${TAG}.err
if [ "$2" == "ncu" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv \
     --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 5 --warmup 2 --no-cpu-baseline > /dev/null 2>&1
  echo "ncu launches rc=$?"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fp_kernel|rle_kernel|rle_sums_kernel|scan_kernel" \
     -s 12 -c 6 -o gpurun_out/prof_${TAG} -f python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/ncu_full_${TAG}.log 2>&1
  echo "ncu full rc=$?"
fi
