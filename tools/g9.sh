mkdir -p gpurun_out/race
for sel in "lz4_overlapping_matches[4]" "corrupt_ans or lz4_overlapping_matches[4]" "corrupt_strdict or lz4_overlapping_matches[4]" "strdict_long or lz4_overlapping_matches[4]" "golden or lz4_overlapping_matches[4]" "config1 or lz4_overlapping_matches[4]"; do
  timeout 600 compute-sanitizer --tool racecheck python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "$sel" > gpurun_out/race/bisect.log 2>&1
  echo "[$sel] rc=$? $(grep -E 'passed|failed' gpurun_out/race/bisect.log | tail -1) $(grep -o 'resident=[A-Za-z]*: offsets' gpurun_out/race/bisect.log | head -1)"
done
