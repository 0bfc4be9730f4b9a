#!/bin/bash
# the round-1 racecheck selection under compute-sanitizer racecheck in five variants (profiles/r02_racecheck.md)
mkdir -p gpurun_out/race
RSEL="golden or config1 or strdict_long or corrupt_strdict or corrupt_ans or lz4_overlapping_matches[1] or lz4_overlapping_matches[4] or dstride_random_runs[3]"
for env in "X=1" "CDM_PDL=0" "CDM_SCAN_MODE=1" "CDM_SERIAL=1" "CDM_SERIAL=1 CDM_PDL=0"; do
  tag=$(echo $env | tr ' =' '__')
  timeout 600 env $env compute-sanitizer --tool racecheck python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "$RSEL" > gpurun_out/race/full_$tag.log 2>&1
  echo "[$env] rc=$? $(grep -E 'passed|failed' gpurun_out/race/full_$tag.log | tail -1) $(grep -o 'resident=[A-Za-z]*: offsets' gpurun_out/race/full_$tag.log | head -1) $(grep FAILED gpurun_out/race/full_$tag.log | head -1)"
done
timeout 900 python -m pytest tests/test_gpu_boundary.py -q -x -p no:cacheprovider > gpurun_out/pytest_boundary.log 2>&1; echo "boundary rc=$?"; tail -15 gpurun_out/pytest_boundary.log
