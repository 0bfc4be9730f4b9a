mkdir -p gpurun_out/race
RSEL="golden or config1 or strdict_long or corrupt_strdict or corrupt_ans or lz4_overlapping_matches[1] or lz4_overlapping_matches[4] or dstride_random_runs[3]"
for env in "X=1" "CDM_PDL=0" "CDM_SCAN_MODE=1" "CDM_SERIAL=1"; do
  timeout 600 env $env compute-sanitizer --tool racecheck python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "$RSEL" > gpurun_out/race/full_$env.log 2>&1
  echo "[$env] rc=$? $(grep -E 'passed|failed' gpurun_out/race/full_$env.log | tail -1) $(grep -o 'resident=[A-Za-z]*: offsets' gpurun_out/race/full_$env.log | head -1) $(grep FAILED gpurun_out/race/full_$env.log | head -1)"
done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "scan or varchar or lz4 or tpch_columns" > gpurun_out/pytest_sel.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_sel.log
timeout 600 python tools/microbench.py SCAN > gpurun_out/mb_scan.txt 2>&1; grep "^|" gpurun_out/mb_scan.txt | tail -7
CDM_SCAN_DIRECT=0 timeout 600 python tools/microbench.py SCAN > gpurun_out/mb_scan_t.txt 2>&1; grep "^|" gpurun_out/mb_scan_t.txt | tail -7
