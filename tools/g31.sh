mkdir -p gpurun_out
CDM_LZ4_DIN=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "lz4 or varchar or l_comment" > gpurun_out/pytest_lz4.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_lz4.log
for d in 0 1; do CDM_LZ4_DIN=$d timeout 600 python tools/microbench.py NP --filter "lz4" > gpurun_out/mb_np_din$d.txt 2>&1; echo "din $d"; grep "^|" gpurun_out/mb_np_din$d.txt | tail -6; done
