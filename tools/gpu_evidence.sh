#!/bin/bash
# one round of evidence: GPU tests, bench lines (config2 headline, reference arm, config3, config4, ans),
# ncu launch list of the headline bench, ncu --set full of one config-2 batch, microbenchmarks
TAG=${1:-r01}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 -p no:cacheprovider > gpurun_out/pytest_${TAG}.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/pytest_${TAG}.log
timeout 600 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; echo "bench rc=$?"
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_${TAG}.json 2>&1
timeout 600 python bench.py --workload config3 --steps 20 --warmup 3 > gpurun_out/bench_config3_${TAG}.json 2>/dev/null
timeout 900 python bench.py --workload config4 --steps 20 --warmup 3 > gpurun_out/bench_config4_${TAG}.json 2>/dev/null
timeout 600 python bench.py --workload ans --steps 20 --warmup 3 > gpurun_out/bench_ans_${TAG}.json 2>/dev/null
timeout 600 python bench.py --workload strdict --steps 10 --warmup 3 > gpurun_out/bench_strdict_${TAG}.json 2>/dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
   --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
echo "ncu launches rc=$?"
CDM_SERIAL=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fp_kernel|rle_kernel|rle_sums|scan_kernel|lz4_|ans_" \
   -c 6 -o gpurun_out/prof_${TAG} -f python tools/one_batch.py 1 config2 > gpurun_out/ncu_full_${TAG}.log 2>&1
echo "ncu full rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sd_|ans_warp" \
   -c 4 -o gpurun_out/prof_sd_${TAG} -f python tools/one_batch.py 1 strdict > gpurun_out/ncu_sd_${TAG}.log 2>&1
echo "ncu strdict rc=$?"
timeout 1500 python tools/microbench.py E2 E3 E7 NP --rows 67108864 --steps 10 > gpurun_out/microbench_${TAG}.txt 2>&1
echo "microbench rc=$?"
timeout 900 python tools/tune.py --steps 5 > gpurun_out/tune_${TAG}.txt 2>&1
echo "tune rc=$?"
