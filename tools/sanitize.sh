#!/bin/bash
# compute-sanitizer memcheck + racecheck (shared-memory hazards) on representative GPU parity tests
mkdir -p gpurun_out
for tool in memcheck racecheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
    python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider \
    -k "golden or config1 or delta_scan_many_tiles[3] or rle_distributions[even-4] or giant or lz4_overlapping or corrupt or tpch_columns and (l_orderkey or l_shipmode or l_comment or o_orderkey or l_returnflag) or corrupt_ans" \
    > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/sanitize_$tool.log
done
