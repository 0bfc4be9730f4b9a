mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.log
timeout 600 python tools/microbench.py CHR SCAN > gpurun_out/mb_chr_scan.txt 2>&1; grep "^|" gpurun_out/mb_chr_scan.txt | tail -14
CDM_SCAN_MODE=1 timeout 600 python tools/microbench.py SCAN > gpurun_out/mb_scan_lb.txt 2>&1; grep "^|" gpurun_out/mb_scan_lb.txt | tail -7
CDM_LZ4_G=1 timeout 600 python tools/microbench.py NP > gpurun_out/mb_np_g1.txt 2>&1; grep "^|" gpurun_out/mb_np_g1.txt | tail -8
