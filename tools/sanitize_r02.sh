#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck on the round-2 kernels (fpc_kernel incl. pre-shifted tables, all three scan schedules, lz4_thread / split / spec kernels, String-dictionary, RLE group sums, multi-link ingestion, engine checksums)
mkdir -p gpurun_out
SEL=${1:-"char_rows_every_width or tpch_columns or bitpack_every_width or delta_scan_many_tiles or varchar_offsets or (lz4 and spec) or lz4_lane_widths or corrupt_lz4 or corrupt_char or golden or strdict or delta_dict or gp_occupancy_knob or rle_zero_length or dstride_random_runs"}
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 20 \
  python -m pytest tests/test_gpu_parity.py tests/test_gpu_boundary.py -q -p no:cacheprovider -k "$SEL or multi_link or checksum_matches" > gpurun_out/r02_sanitize_memcheck.log 2>&1
echo "memcheck rc=$?"; tail -3 gpurun_out/r02_sanitize_memcheck.log
timeout 1500 compute-sanitizer --tool racecheck --error-exitcode 9 --print-limit 20 \
  python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "$SEL" > gpurun_out/r02_sanitize_racecheck.log 2>&1
echo "racecheck rc=$?"; tail -3 gpurun_out/r02_sanitize_racecheck.log
timeout 1500 compute-sanitizer --tool synccheck --error-exitcode 9 --print-limit 20 \
  python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "$SEL" > gpurun_out/r02_sanitize_synccheck.log 2>&1
echo "synccheck rc=$?"; tail -3 gpurun_out/r02_sanitize_synccheck.log
