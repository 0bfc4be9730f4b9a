mkdir -p gpurun_out/race
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "lz4" > gpurun_out/pytest_lz4.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_lz4.log
CDM_LZ4_G=1 timeout 600 python tools/microbench.py NP --filter lz4 > gpurun_out/mb_np_g1.txt 2>&1; grep "^|" gpurun_out/mb_np_g1.txt | tail -3
ncu --set full --import-source on -k regex:scan_kernel_rts --launch-count 1 -o gpurun_out/scan_rts2 -f python tools/microbench.py SCAN --filter "config1 sorted" --steps 1 > gpurun_out/ncu_scan.log 2>&1; tail -1 gpurun_out/ncu_scan.log
RSEL="golden or config1 or strdict_long or corrupt_strdict or corrupt_ans or lz4_overlapping_matches[1] or lz4_overlapping_matches[4] or dstride_random_runs[3]"
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "$RSEL" > gpurun_out/race/suite_rc_rts.log 2>&1; echo "rts rc=$?"; tail -3 gpurun_out/race/suite_rc_rts.log
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python tools/race_probe.py --parity --scan-mode 1 --lanes 4 --replays 6 > gpurun_out/race/probe_parity_lb.log 2>&1; echo "probe lb rc=$?"; grep -E "mode|replay|probe|SUMMARY" gpurun_out/race/probe_parity_lb.log | head -14
