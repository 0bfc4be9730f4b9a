mkdir -p gpurun_out
ncu --set full --import-source on -k regex:lz4_thread --launch-count 1 -o gpurun_out/lz4_thread3 -f python tools/microbench.py NP --filter "sub=16384" --steps 1 > gpurun_out/ncu_lz4.log 2>&1; tail -1 gpurun_out/ncu_lz4.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "scan or varchar or lz4 or tpch_columns or empty or delta" > gpurun_out/pytest_sel.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_sel.log
timeout 600 python tools/microbench.py SCAN > gpurun_out/mb_scan.txt 2>&1; grep "^|" gpurun_out/mb_scan.txt | tail -7
