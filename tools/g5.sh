mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "lz4 or scan or varchar or tpch_columns or empty" > gpurun_out/pytest_sel.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_sel.log
timeout 600 python tools/microbench.py SCAN > gpurun_out/mb_scan.txt 2>&1; grep "^|" gpurun_out/mb_scan.txt | tail -7
CDM_LZ4_G=1 timeout 600 python tools/microbench.py NP > gpurun_out/mb_np_g1.txt 2>&1; grep "^|" gpurun_out/mb_np_g1.txt | tail -8
