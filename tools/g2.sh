set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "char_rows or tpch_columns" > gpurun_out/char_tests.log 2>&1; tail -3 gpurun_out/char_tests.log
timeout 600 python tools/microbench.py CHR > gpurun_out/chr_new.txt 2>&1; tail -9 gpurun_out/chr_new.txt
CDM_FPC=0 timeout 600 python tools/microbench.py CHR > gpurun_out/chr_old.txt 2>&1; tail -9 gpurun_out/chr_old.txt
RSEL="golden or config1 or strdict_long or corrupt_strdict or corrupt_ans or lz4_overlapping_matches[1] or lz4_overlapping_matches[4] or dstride_random_runs[3]"
timeout 1500 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "$RSEL" > gpurun_out/race/suite_rc.log 2>&1; echo "rc=$?"; tail -30 gpurun_out/race/suite_rc.log
