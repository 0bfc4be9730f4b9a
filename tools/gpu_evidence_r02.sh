#!/bin/bash
# round-2 evidence: ncu --set full of the config-4 LZ4 launch (traffic per launch), launch list of the headline bench
TAG=${1:-r02q}
mkdir -p gpurun_out
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:lz4_thread -c 1 -o gpurun_out/c4_lz4_${TAG} -f \
  python tools/one_batch.py 1 config4 > gpurun_out/ncu_c4lz4_${TAG}.log 2>&1
echo "ncu full rc=$?"; tail -2 gpurun_out/ncu_c4lz4_${TAG}.log
python tools/ncu_traffic.py gpurun_out/c4_lz4_${TAG}.ncu-rep profiles/ncu_traffic.json --key=config4:lz4_thread_kernel
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/launches_${TAG}.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launches_${TAG}.log 2>&1
echo "ncu launches rc=$?"
