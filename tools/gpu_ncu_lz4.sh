#!/bin/bash
# ncu --set full (source-level) of one launch of the LZ4 kernel in a microbench case
TAG=${1:-lz4}; FILT=${2:-"one sub-chunk sub=16384"}; KREG=${3:-lz4_spec}
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$KREG" -s 1 -c 1 -o gpurun_out/ncu_${TAG} -f \
  python tools/microbench.py NP --filter "$FILT" --steps 2 > gpurun_out/ncu_${TAG}.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/ncu_${TAG}.log
