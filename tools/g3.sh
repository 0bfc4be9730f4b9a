mkdir -p gpurun_out/race
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python tools/microbench.py CHR SCAN > gpurun_out/mb_chr_scan.txt 2>&1; tail -16 gpurun_out/mb_chr_scan.txt
RSEL="golden or config1 or strdict_long or corrupt_strdict or corrupt_ans or lz4_overlapping_matches[1] or lz4_overlapping_matches[4] or dstride_random_runs[3]"
timeout 1500 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "$RSEL" > gpurun_out/race/suite_rc.log 2>&1; echo "rc=$?"; tail -30 gpurun_out/race/suite_rc.log
