#!/bin/bash
# compute-sanitizer memcheck + racecheck (shared-memory hazards) on representative GPU parity tests
mkdir -p gpurun_out
SEL=${1:-"golden or config1 or delta_scan_many_tiles[3] or rle_distributions[even-4] or giant or lz4_overlapping or corrupt or tpch_columns and (l_orderkey or l_shipmode or l_comment or o_orderkey or l_returnflag or o_comment) or dstride or strdict or checksum or lz4_lane_widths"}
RSEL=${2:-"golden or config1 or strdict_long or corrupt_strdict or corrupt_ans or lz4_overlapping_matches[1] or lz4_overlapping_matches[4] or dstride_random_runs[3]"}
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 20 \
  python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "$SEL" > gpurun_out/sanitize_memcheck.log 2>&1
echo "memcheck rc=$?"; tail -3 gpurun_out/sanitize_memcheck.log
timeout 1500 compute-sanitizer --tool racecheck --error-exitcode 9 --print-limit 20 \
  python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "$RSEL" > gpurun_out/sanitize_racecheck.log 2>&1
echo "racecheck rc=$?"; tail -3 gpurun_out/sanitize_racecheck.log
