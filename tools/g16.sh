mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_boundary.py -q -x -p no:cacheprovider -k "scan or varchar or tpch_columns or delta or concurrent or ticket or checksum" > gpurun_out/pytest_sel.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_sel.log
timeout 600 python tools/microbench.py SCAN > gpurun_out/mb_scan.txt 2>&1; grep "^|" gpurun_out/mb_scan.txt | tail -7
timeout 600 python bench.py --workload config5 --sf 10 --steps 2 --warmup 1 > gpurun_out/c5_sf10.log 2>&1; echo "c5 rc=$?"; tail -c 2500 gpurun_out/c5_sf10.log
