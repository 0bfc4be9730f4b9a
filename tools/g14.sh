mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "lz4 or varchar or empty" > gpurun_out/pytest_lz4.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_lz4.log
for m in 3 4; do CDM_LZ4_MINB=$m timeout 600 python tools/microbench.py NP --filter lz4 > gpurun_out/mb_np_$m.txt 2>&1; echo "minb $m"; grep "^|" gpurun_out/mb_np_$m.txt | tail -3; done
