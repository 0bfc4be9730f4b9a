mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_gpu.log
timeout 600 python tools/microbench.py SCAN CHR > gpurun_out/mb_scan_chr.txt 2>&1; grep "^|" gpurun_out/mb_scan_chr.txt | tail -13
CDM_SCAN_MODE=1 timeout 600 python tools/microbench.py SCAN > gpurun_out/mb_scan_lb.txt 2>&1; grep "^|" gpurun_out/mb_scan_lb.txt | tail -7
